"""Full-size parity on BASELINE configs c2 (10K^3, 1e8 nnz, R=16, Poisson,
p = q = 1e7) and c3 (5-way LBNL-shaped, 1.7e6 nnz, u128 keys, R=10,
Bernoulli, p = q = 1e6; the L2 Bloom filter is in front of its hash), and a
c4-shaped tensor scaled to 1e8 nonzeros (Amazon dims 4.8M x 1.8M x 1.8M, R=16,
Gaussian, p = q = 1e7): its 538 MB of factors spill L2, so the layout c4 and
c5 run by default -- A/G rows interleaved, slots visited in mode-1 order, no
filter -- is the one under test; and a c5-shaped one (Reddit dims, R=32,
Poisson, 1e8 nonzeros, p = q = 1e7: 128-B rows, 8 lanes per sample).  All in the launch configuration bench.py
times: sampled slots bit-exact (first 1e5 slots of each stratum + 100 random
windows of 1000), the full-size gradient element-wise against the oracle's
fp64 fused sampling-MTTKRP over all p + q samples, and the loss estimate at the
config's f.  Plus, on c2, the sampler's distribution at scale:
the mean of 100 GPU gradients against the exact Poisson gradient.  Heavy
(several minutes of oracle host time)."""
import numpy as np
import pytest
import torch

import gcp_synth

pytestmark = pytest.mark.gpu


# c4's shape and loss at c2's size: the DRAM-resident-factor layout at a size
# the oracle still sorts (SURVEY C18 asks c2-c5 index parity)
C4S = dict(gcp_synth.CONFIGS["c4"], nnz=100_000_000)
# c5's shape, R = 32 and loss at the same size (p = q = 1e7): 128-B rows (8 lanes
# per sample), 2.1 GB of factors, no A/G interleave (rows fill a line alone)
C5S = dict(gcp_synth.CONFIGS["c5"], nnz=100_000_000, s=10_000_000, f=10_000_000)


@pytest.fixture(scope="module", params=["c2", "c3", "c4s", "c5s"])
def full(orc, request):
    import paper_2605_20353_b200 as g
    if request.param == "c4s":
        cfg, seeds = C4S, gcp_synth.SEEDS["c4"]
    elif request.param == "c5s":
        cfg, seeds = C5S, gcp_synth.SEEDS["c5"]
    else:
        cfg, seeds = gcp_synth.CONFIGS[request.param], gcp_synth.SEEDS[request.param]
    subs, vals = gcp_synth.chi_kolda(cfg["dims"], cfg["nnz"], cfg["R"], seeds["data"], cfg["loss"], device="cuda")
    subs_h, vals_h = subs.cpu().numpy(), vals.cpu().numpy()
    del subs, vals
    torch.cuda.empty_cache()
    ctx = g.Context(0, None, "fp32")
    ctx.tensor_create(cfg["dims"], subs_h, vals_h)
    ctx.model_init(cfg["R"], seeds["model"])
    if cfg["loss"] == "bernoulli":   # centre the model so sigma(m) is not saturated (as the parity tests do)
        for k in range(len(cfg["dims"])):
            ctx.model_set(k, ctx.model_get(k) - 0.5)
    ctx.sample("stratified", cfg["s"], cfg["s"], seeds["sample"])
    lay = ctx.layout()
    if request.param == "c4s":   # the bench's DRAM-resident layout, chosen by default (no env forcing)
        assert lay["ag_interleaved"] and lay["slot_order"], lay
    elif request.param == "c5s":  # 128-B rows: no interleave; 2e7 slots: ordered (full c5's 2e8 are not)
        assert not lay["ag_interleaved"] and lay["slot_order"], lay
    else:
        assert not lay["ag_interleaved"] and not lay["slot_order"], lay
    t = orc.Tensor(cfg["dims"], subs_h, vals_h)
    return ctx, t, cfg, seeds, (subs_h, vals_h)


def test_full_size_sample_indices_bit_exact(orc, full):
    ctx, t, cfg, seeds, _ = full
    p = cfg["s"]
    rng = np.random.default_rng(0)
    for stratum in (0, 1):
        gs, gj, gw, ga = ctx.sample_export(stratum, 0, 100_000)
        os_, oj, ow, oa = orc.sample_export(t, stratum, seeds["sample"], 0, 0, p, 0, 100_000)
        assert np.array_equal(gs, os_) and np.array_equal(gj, oj) and np.array_equal(ga, oa)
        assert np.array_equal(gw, ow)
        for first in rng.integers(0, p - 1000, size=100):
            gs, gj, _, ga = ctx.sample_export(stratum, int(first), 1000)
            os_, oj, _, oa = orc.sample_export(t, stratum, seeds["sample"], 0, 0, p, int(first), 1000)
            assert np.array_equal(gs, os_) and np.array_equal(gj, oj) and np.array_equal(ga, oa)


def test_full_size_gradient_and_loss_estimate(orc, full):
    ctx, t, cfg, seeds, _ = full
    d = len(cfg["dims"])
    A = [ctx.model_get(k) for k in range(d)]
    ctx.loss_grad(cfg["loss"])
    G = [ctx.grad_get(k) for k in range(d)]
    Go, S, _ = orc.sampled_grad(t, A, cfg["loss"], seeds["sample"], 0, 0, cfg["s"], cfg["s"])
    for k in range(d):
        diff = np.abs(G[k] - Go[k])
        assert (diff <= 1e-4 * S[k]).all(), f"mode {k}: worst {(diff / S[k]).max():.2e}"
        assert np.linalg.norm(G[k] - Go[k]) <= 1e-4 * np.linalg.norm(Go[k])
    est = ctx.loss_estimate(cfg["loss"], cfg["f"], cfg["f"], 2)
    oe, sc = orc.loss_estimate(t, A, cfg["loss"], 2, 0, cfg["f"], cfg["f"])
    assert abs(est - oe) <= 1e-4 * sc


def test_sampler_distribution_at_scale(orc, full):
    """SURVEY C17 "GPU sampler distribution at scale": independent of the
    oracle's sampling stream, the mean of K = 100 GPU sampled gradients (seeds
    3002 + k, fresh iteration words) on c2 converges to the exact gradient
    dF/dA of the Poisson objective (closed form over all 1e12 entries,
    oracle.poisson_exact_grad): per mode ||mean - exact||_F <= 3 ||SE||_F,
    SE the per-element standard error of the mean (unbiased weights)."""
    ctx, t, cfg, seeds, (subs_h, vals_h) = full
    if cfg is not gcp_synth.CONFIGS["c2"]:
        # c5s (Poisson too) passed the 3-SE check, but its zero weight (M - N)/q
        # ~ 1.2e12 at q = 1e7 leaves each gradient ~1.2x its own size in noise
        # (SE of the 100-mean 12% of the gradient), and the 100 gradient reads
        # of 2 GB each cost ~12 min (profiles/r02z_tests.log): c2 only
        pytest.skip("sampler distribution at scale: c2")
    d, K = len(cfg["dims"]), 100
    A = [ctx.model_get(k) for k in range(d)]
    exact = orc.poisson_exact_grad(subs_h, vals_h, A)
    acc = [np.zeros_like(a) for a in A]
    sq = [np.zeros_like(a) for a in A]
    import paper_2605_20353_b200 as g
    zero_step = g.adam_params(rate=0.0)   # resets G, leaves A (rate 0), advances the iteration word
    ctx.loss_grad(cfg["loss"])            # (a gradient left by another test is dropped with it)
    ctx.adam_step(zero_step)
    for k in range(K):
        ctx.sample("stratified", cfg["s"], cfg["s"], 3002 + k)
        ctx.loss_grad(cfg["loss"])
        for m in range(d):
            Gm = ctx.grad_get(m)
            acc[m] += Gm
            sq[m] += Gm * Gm
        ctx.adam_step(zero_step)
    for m in range(d):
        assert np.array_equal(ctx.model_get(m), A[m])
        mean = acc[m] / K
        se = np.sqrt(np.maximum(sq[m] / K - mean ** 2, 0) / (K - 1))
        err, bound = np.linalg.norm(mean - exact[m]), 3 * np.linalg.norm(se)
        assert err <= bound, f"mode {m}: |mean - exact| = {err:.4g} > 3 SE = {bound:.4g}"
        # and the estimator is not trivially noisy: SE well below the gradient's size
        assert np.linalg.norm(se) < 0.05 * np.linalg.norm(exact[m])
