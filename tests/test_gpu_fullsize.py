"""Full-size parity on BASELINE configs c2 (10K^3, 1e8 nnz, R=16, Poisson,
p = q = 1e7) and c3 (5-way LBNL-shaped, 1.7e6 nnz, u128 keys, R=10,
Bernoulli, p = q = 1e6; the L2 Bloom filter is in front of its hash) in the
launch configuration bench.py times: sampled slots are compared bit-exactly
(first 1e5 slots of each stratum + 1e5 random slots), the full-size gradient
element-wise against the oracle's fp64 fused sampling-MTTKRP over all p + q
samples, and the loss estimate at the config's f.  Heavy (about 2-3 minutes of
oracle host time for c2)."""
import numpy as np
import pytest
import torch

import gcp_synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["c2", "c3"])
def full(orc, request):
    import paper_2605_20353_b200 as g
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
    t = orc.Tensor(cfg["dims"], subs_h, vals_h)
    return ctx, t, cfg, seeds


def test_full_size_sample_indices_bit_exact(orc, full):
    ctx, t, cfg, seeds = full
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
    ctx, t, cfg, seeds = full
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
