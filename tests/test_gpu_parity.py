"""GPU parity: libgcp.so (through the C ABI) against the fp64 oracle.

Bit-exact: sample coordinates, nonzero indices j, attempt counts, canonical
order, hash membership, factor initialisation (fp32 = round(fp64)).
Tolerance: gradients per element |dG| <= tol * S (S = the
oracle's rounding-scale sum) and per mode ||dG||_F <= tol ||G||_F, with
tol = 1e-4 (fp32) / 1e-10 (fp64); loss estimates |dF| <= tol * sum|terms|.
"""
import math

import numpy as np
import pytest

import gcp_synth

pytestmark = pytest.mark.gpu

LOSSES = ["gaussian", "poisson", "bernoulli"]
TOL = {"fp32": 1e-4, "fp64": 1e-10}


@pytest.fixture(scope="module")
def gcp():
    import paper_2605_20353_b200 as g
    return g


def _tensor(loss, dims=(20, 30, 40), nnz=2400, seed=1001):
    subs, vals = gcp_synth.chi_kolda(dims, nnz, 4, seed, loss=loss)
    subs, vals = subs.numpy(), vals.numpy()
    if loss == "gaussian":
        vals = vals - 1.5  # signed data
    return subs, vals


def _ctx(gcp, dims, subs, vals, prec="fp32", R=4, mseed=2001):
    c = gcp.Context(0, None, prec)
    c.tensor_create(dims, subs, vals)
    c.model_init(R, mseed)
    return c


def _model(c, d):
    return [c.model_get(k) for k in range(d)]


def test_canonical_order_and_membership(gcp, orc):
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals)
    t = orc.Tensor(dims, subs, vals)
    ss, sv = t.sorted()
    gs, gv = c.tensor_export_sorted(0, len(vals))
    assert np.array_equal(gs, ss) and np.array_equal(gv, sv.astype(np.float32).astype(np.float64))
    assert c.tensor_contains(subs).all()
    rng = np.random.default_rng(0)
    cand = np.stack([rng.integers(0, I, 20000) for I in dims], 1)
    want = np.array([t.contains(x) for x in cand])
    assert np.array_equal(c.tensor_contains(cand), want)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_factor_init_bit_exact(gcp, orc, prec):
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals, prec=prec, R=5)
    A = orc.factor_init(2001, dims, 5)
    for k in range(3):
        want = A[k].astype(np.float32).astype(np.float64) if prec == "fp32" else A[k]
        assert np.array_equal(c.model_get(k), want)


@pytest.mark.parametrize("strategy", ["stratified", "semi"])
def test_sample_indices_bit_exact(gcp, orc, strategy):
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals)
    t = orc.Tensor(dims, subs, vals)
    p, q = 1000, 1000
    for it in range(3):
        c.sample(strategy, p, q, 3001)
        for stratum, n in ((0, p), (1, q)):
            gs, gj, gw, ga = c.sample_export(stratum, 0, n)
            os_, oj, ow, oa = orc.sample_export(t, stratum, 3001, 0, it, n, 0, n, strategy=strategy)
            assert np.array_equal(gs, os_)
            assert np.array_equal(gj, oj)
            assert np.array_equal(ga, oa)
            assert np.array_equal(gw, ow)
        if stratum == 1 and strategy == "stratified":
            assert oa.max() > 1  # rejection really fired at rho = 0.1
        # advance the iteration counter (it) by one Adam step
        c.loss_grad("poisson")
        c.adam_step()


def _grad_check(G, Go, S, tol, label):
    for k, (g, go, s) in enumerate(zip(G, Go, S)):
        diff = np.abs(g - go)
        bad = diff > tol * s + 1e-300
        assert not bad.any(), f"{label} mode {k}: {bad.sum()} elements, worst {diff[bad].max()} vs {s[bad].max()}"
        assert np.linalg.norm(g - go) <= tol * np.linalg.norm(go) + 1e-300, label


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("strategy", ["stratified", "semi"])
@pytest.mark.parametrize("loss", LOSSES)
def test_gradient_parity(gcp, orc, loss, strategy, prec):
    dims = (20, 30, 40)
    subs, vals = _tensor(loss)
    c = _ctx(gcp, dims, subs, vals, prec=prec)
    if loss == "bernoulli":  # centre the model so sigma(m) is not saturated
        for k in range(3):
            c.model_set(k, c.model_get(k) - 0.5)
    t = orc.Tensor(dims, subs, vals)
    p, q = 1000, 1000
    c.sample(strategy, p, q, 3001)
    A = _model(c, 3)
    ls = c.loss_grad(loss, want_loss=True)
    G = [c.grad_get(k) for k in range(3)]
    Go, S, lo, lsc = orc.sampled_grad(t, A, loss, 3001, 0, 0, p, q, strategy, loss_scale=True)
    _grad_check(G, Go, S, TOL[prec], f"{loss}/{strategy}/{prec}")
    # sampled loss sum_s w f: C18, |dF| <= tol * sum |terms| (rounding scales of f)
    assert abs(ls - lo) <= TOL[prec] * lsc, (ls, lo, lsc, abs(ls - lo) / lsc)


@pytest.mark.parametrize("interleave", ["0", "1"])
def test_ag_layouts_agree(gcp, orc, interleave, monkeypatch):
    """Separate and row-interleaved A/G layouts: same gradient, same Adam step."""
    monkeypatch.setenv("GCP_AG_INTERLEAVE", interleave)
    dims = (20, 30, 40)
    subs, vals = _tensor("gaussian")
    c = _ctx(gcp, dims, subs, vals, prec="fp64")
    t = orc.Tensor(dims, subs, vals)
    c.sample("stratified", 700, 900, 3001)
    A = _model(c, 3)
    c.loss_grad("gaussian")
    G = [c.grad_get(k) for k in range(3)]
    Go, S, _ = orc.sampled_grad(t, A, "gaussian", 3001, 0, 0, 700, 900)
    _grad_check(G, Go, S, 1e-10, f"interleave={interleave}")
    c.adam_step(gcp.adam_params(rate=1e-2))
    flat = np.concatenate([a.ravel() for a in A])
    Gf = np.concatenate([g.ravel() for g in Go])
    orc.adam(flat, Gf, np.zeros_like(flat), np.zeros_like(flat), 1, 1e-2, 0.9, 0.999, 1e-8)
    got = np.concatenate([a.ravel() for a in _model(c, 3)])
    assert np.allclose(got, flat, rtol=1e-9, atol=1e-12)
    assert all((c.grad_get(k) == 0).all() for k in range(3))   # G reset fused into Adam


@pytest.mark.parametrize("tiles", ["1", "many"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("strategy", ["stratified", "semi"])
def test_slot_order_same_gradient(gcp, orc, strategy, prec, tiles, monkeypatch):
    """GCP_SLOT_ORDER=1: the gradient K2 visits its slots grouped by mode-1
    position (histogram / scan / scatter of the slots, kernels.cu; "many": the
    slots ordered in independent tiles of 1024, the layout large p + q take).
    Same sample set, so the same gradient as the oracle's within the fp
    tolerance; p + q spans many warps and a ragged tail."""
    monkeypatch.setenv("GCP_SLOT_ORDER", "1")
    if tiles == "many":
        monkeypatch.setenv("GCP_ORD_TILE_MB", "0.001")
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals, prec=prec)
    t = orc.Tensor(dims, subs, vals)
    for it, (p, q) in enumerate([(1000, 1000), (3333, 77), (0, 1501)]):
        c.sample(strategy, p, q, 3001)
        A = _model(c, 3)
        c.loss_grad("poisson")
        G = [c.grad_get(k) for k in range(3)]
        Go, S, _ = orc.sampled_grad(t, A, "poisson", 3001, 0, it, p, q, strategy)
        _grad_check(G, Go, S, TOL[prec], f"slot order {strategy}/{prec} p={p} q={q}")
        c.adam_step(gcp.adam_params(rate=1e-2))   # resets G, advances the iteration counter


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("R", [4, 10, 16, 40])
@pytest.mark.parametrize("order", ["0", "1"])
def test_warp_aggregated_scatter_same_gradient(gcp, orc, prec, R, order, monkeypatch):
    """GCP_WAGG=1: the samples of a K2 round that hit the same row of a mode
    sum their contributions in registers (__match_any_sync) and one group
    issues the red.add (P:591-598's atomic MTTKRP, aggregated).  20/30/40 rows
    make repeats frequent (R = 4: 32 samples per round); R = 10 leaves a lane
    of every group without a vector (the shuffles must still include it);
    R = 40 two vectors per lane.  Same samples, so the oracle's gradient within
    the C18 tolerance, slot order on and off."""
    monkeypatch.setenv("GCP_WAGG", "1")
    monkeypatch.setenv("GCP_SLOT_ORDER", order)
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals, prec=prec, R=R)
    t = orc.Tensor(dims, subs, vals)
    for it, (p, q) in enumerate([(1000, 1000), (3333, 77)]):
        c.sample("stratified", p, q, 3001)
        A = _model(c, 3)
        c.loss_grad("poisson")
        G = [c.grad_get(k) for k in range(3)]
        Go, S, _ = orc.sampled_grad(t, A, "poisson", 3001, 0, it, p, q, "stratified")
        _grad_check(G, Go, S, TOL[prec], f"wagg R={R} {prec} order={order} p={p} q={q}")
        c.adam_step(gcp.adam_params(rate=1e-2))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("loss", LOSSES)
def test_loss_estimate_parity(gcp, orc, loss, prec):
    dims = (20, 30, 40)
    subs, vals = _tensor(loss)
    c = _ctx(gcp, dims, subs, vals, prec=prec)
    t = orc.Tensor(dims, subs, vals)
    A = _model(c, 3)
    est = c.loss_estimate(loss, 2000, 2000, 4001)
    oe, scale = orc.loss_estimate(t, A, loss, 4001, 0, 2000, 2000)
    assert abs(est - oe) <= TOL[prec] * scale


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_adam_parity_from_identical_gradient(gcp, orc, prec):
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals, prec=prec)
    c.sample("stratified", 1000, 1000, 3001)
    A = np.concatenate([a.ravel() for a in _model(c, 3)])
    B = np.zeros_like(A)
    Cm = np.zeros_like(A)
    for step in range(1, 4):
        c.loss_grad("poisson")
        G = np.concatenate([c.grad_get(k).ravel() for k in range(3)])
        p = gcp.adam_params(rate=1e-2, beta1=0.9, beta2=0.999, eps=1e-8)
        c.adam_step(p)
        orc.adam(A, G, B, Cm, step, 1e-2, 0.9, 0.999, 1e-8, 0.0)
        Ag = np.concatenate([a.ravel() for a in _model(c, 3)])
        # C18: elementwise relative tol with an absolute floor tol * alpha
        tol, alpha = TOL[prec], 1e-2
        err = np.abs(Ag - A)
        assert np.all(err <= tol * np.abs(A) + tol * alpha), (step, (err / (tol * np.abs(A) + tol * alpha)).max())
        A = Ag.copy()  # continue from the GPU state (identical-state protocol, C18)
        assert (Ag >= 0).all()  # Poisson clamp l = 0
    ctr = c.counters()
    assert ctr["it"] == 3 and ctr["t"] == 3


def test_zero_gradient_and_errors(gcp):
    dims = (2, 2, 2)
    full = np.array(np.unravel_index(np.arange(8), dims)).T
    c = gcp.Context(0, None, "fp32")
    with pytest.raises(gcp.GcpError) as e:
        c.tensor_create(dims, np.array([[0, 0, 0], [0, 0, 0]]), np.array([1.0, 2.0]))
    assert e.value.name == "GCP_E_DUP"
    with pytest.raises(gcp.GcpError) as e:
        c.tensor_create(dims, np.array([[0, 2, 0]]), np.array([1.0]))
    assert e.value.name == "GCP_E_RANGE"
    with pytest.raises(gcp.GcpError) as e:
        c.tensor_create(dims, np.array([[0, 1, 0]]), np.array([np.inf]))
    assert e.value.name == "GCP_E_ARG"
    c.tensor_create(dims, full, np.ones(8))
    with pytest.raises(gcp.GcpError) as e:
        c.sample("stratified", 10, 10, 1)
    assert e.value.name == "GCP_E_NO_ZEROS"
    with pytest.raises(gcp.GcpError) as e:
        c.loss_grad("poisson")
    assert e.value.name == "GCP_E_STATE"
    # a failed replacement leaves the context without a tensor (the old one is freed first)
    with pytest.raises(gcp.GcpError):
        c.tensor_create(dims, np.array([[0, 0, 0], [0, 0, 0]]), np.array([1.0, 2.0]))
    with pytest.raises(gcp.GcpError) as e:
        c.sample("stratified", 10, 10, 1)
    assert e.value.name == "GCP_E_STATE"
    # one zero in 10^4 entries: the rejection cap fires (reading R5) and is sticky
    dims = (10, 10, 100)
    lin = np.arange(10 * 10 * 100)[1:]
    c2 = gcp.Context(0, None, "fp32")
    c2.tensor_create(dims, np.array(np.unravel_index(lin, dims)).T, np.ones(len(lin)))
    c2.model_init(2, 1)
    c2.sample("stratified", 10, 10, 1)
    with pytest.raises(gcp.GcpError) as e:
        c2.loss_grad("poisson", want_loss=True)
    assert e.value.name == "GCP_E_REJECT_CAP"
    with pytest.raises(gcp.GcpError) as e:
        c2.model_get(0)
    assert e.value.name == "GCP_E_STATE"


def test_u128_keys_lbnl_shape(gcp, orc):
    """c3's 5-way shape has M = 4.0e19 > 2^64: 128-bit keys on the device."""
    dims = gcp_synth.CONFIGS["c3"]["dims"]
    assert math.prod(dims) > 2 ** 64
    rng = np.random.default_rng(5)
    n = 20000
    subs = np.unique(np.stack([rng.integers(0, I, n) for I in dims], 1), axis=0)
    vals = np.ones(len(subs))
    c = _ctx(gcp, dims, subs, vals, R=10)
    t = orc.Tensor(dims, subs, vals)
    assert c.tensor_contains(subs).all()
    cand = np.stack([rng.integers(0, I, 5000) for I in dims], 1)
    cand[:2000] = subs[:2000]
    assert np.array_equal(c.tensor_contains(cand), np.array([t.contains(x) for x in cand]))
    c.sample("stratified", 3000, 3000, 3003)
    for stratum in (0, 1):
        gs, gj, _, ga = c.sample_export(stratum, 0, 3000)
        os_, oj, _, oa = orc.sample_export(t, stratum, 3003, 0, 0, 3000, 0, 3000)
        assert np.array_equal(gs, os_) and np.array_equal(gj, oj) and np.array_equal(ga, oa)
    A = _model(c, 5)
    for k in range(5):
        c.model_set(k, A[k] - 0.4)
    A = _model(c, 5)
    c.loss_grad("bernoulli")
    G = [c.grad_get(k) for k in range(5)]
    Go, S, _ = orc.sampled_grad(t, A, "bernoulli", 3003, 0, 0, 3000, 3000)
    _grad_check(G, Go, S, 1e-4, "u128 bernoulli")


@pytest.mark.parametrize("shape", ["c1", "lbnl"])
def test_sorted_membership_same_draws(gcp, orc, shape):
    """Row f4: the binary-search zero test gives the same samples as the hash set."""
    if shape == "c1":
        dims = (20, 30, 40)
        subs, vals = _tensor("poisson")
        R = 4
    else:
        dims = gcp_synth.CONFIGS["c3"]["dims"]
        rng = np.random.default_rng(6)
        subs = np.unique(np.stack([rng.integers(0, I, 20000) for I in dims], 1), axis=0)
        vals = np.ones(len(subs))
        R = 10
    t = orc.Tensor(dims, subs, vals)
    c = gcp.Context(0, None, "fp32")
    c.set_membership("sorted")
    c.tensor_create(dims, subs, vals)
    c.model_init(R, 2001)
    assert c.tensor_contains(subs).all()
    rng = np.random.default_rng(1)
    cand = np.stack([rng.integers(0, I, 4000) for I in dims], 1)
    cand[:1000] = subs[:1000]
    assert np.array_equal(c.tensor_contains(cand), np.array([t.contains(x) for x in cand]))
    c.sample("stratified", 2000, 2000, 3001)
    gs, gj, _, ga = c.sample_export(1, 0, 2000)
    os_, oj, _, oa = orc.sample_export(t, 1, 3001, 0, 0, 2000, 0, 2000)
    assert np.array_equal(gs, os_) and np.array_equal(ga, oa)
    A = _model(c, len(dims))
    loss = "poisson" if shape == "c1" else "bernoulli"
    c.loss_grad(loss)
    G = [c.grad_get(k) for k in range(len(dims))]
    Go, S, _ = orc.sampled_grad(t, A, loss, 3001, 0, 0, 2000, 2000)
    _grad_check(G, Go, S, 1e-4, "sorted membership")


@pytest.mark.parametrize("graphs,interleave,order", [("1", "0", "0"), ("0", "0", "0"), ("1", "1", "0"),
                                                   ("1", "1", "1")])
def test_fit_matches_oracle(gcp, orc, graphs, interleave, order, monkeypatch):
    """The epoch loop (annealing, R20) against oracle.fit, fp64, on a side
    stream: with GCP_GRAPHS=1 each epoch's iterations replay as one CUDA graph
    with the step state on the device; with 0 they launch one by one; and the
    graph path with A/G rows interleaved (the layout c4 uses), also with the
    slots visited in mode-1 order (captured prepass + radix sort)."""
    import torch
    monkeypatch.setenv("GCP_GRAPHS", graphs)
    monkeypatch.setenv("GCP_AG_INTERLEAVE", interleave)
    monkeypatch.setenv("GCP_SLOT_ORDER", order)
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    stream = torch.cuda.Stream(0)
    c = gcp.Context(0, stream.cuda_stream, "fp64")
    c.tensor_create(dims, subs, vals)
    c.model_init(4, 2001)
    A0 = _model(c, 3)
    kw = dict(epochs=6, max_fails=3, decay=0.1, s_nz=300, s_z=300, f_nz=1500, f_z=1500, seed=7, fseed=2,
              rate=0.3)
    p = c.fit_params(iters_per_epoch=10, loss="poisson", **kw)
    best, rows = c.fit(p)
    blocks, grid = orc.split_blocks(dims, subs, vals, 1)
    Af, hist, obest = orc.fit(blocks, grid, A0, "poisson", iters=10, **kw)
    assert len(rows) == len(hist)
    for (_, _, est, rate, _), (oest, orate, _) in zip(rows, hist):
        assert est == pytest.approx(oest, rel=1e-9)
    assert [r[3] for r in rows] == pytest.approx([h[1] * (1.0 if h[2] else kw["decay"]) for h in hist])
    assert best == pytest.approx(obest, rel=1e-9)
    for k in range(3):
        assert np.allclose(c.model_get(k), Af[k], rtol=1e-8, atol=1e-10)
    cnt = c.counters()
    assert cnt["it"] == 10 * len(rows)   # t rolls back with a rejected epoch, it does not
    assert cnt["t"] == 10 * sum(h[2] for h in hist)


def test_fit_runs_and_decreases(gcp, orc):
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals)
    t = orc.Tensor(dims, subs, vals)
    A0 = _model(c, 3)
    F0, _ = orc.loss_estimate(t, A0, "poisson", 2, 0, 2000, 2000)
    p = c.fit_params(epochs=5, iters_per_epoch=20, s_nz=500, s_z=500, f_nz=2000, f_z=2000, loss="poisson",
                     seed=7, fseed=2, rate=1e-2)
    best, rows = c.fit(p)
    assert len(rows) >= 3
    assert best < F0
    ests = [r[2] for r in rows]
    assert min(ests) == pytest.approx(best)


@pytest.mark.parametrize("membership", ["hash", "sorted"])
def test_filter_leaves_samples_unchanged(gcp, monkeypatch, membership):
    """The L2 Bloom filter in front of the zero test is a pure accelerator: with
    and without it (GCP_FILTER=1/0 at ingest) the zero samples, their
    attempt counts (c1 is dense: rejections happen) and the gradient agree
    bit for bit (gradient: same samples, same kernel; fp64 so atomics order
    cannot blur a difference at this size)."""
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    out = []
    for f in ("1", "0"):
        monkeypatch.setenv("GCP_FILTER", f)
        c = gcp.Context(0, None, "fp64")
        c.set_membership(membership)
        c.tensor_create(dims, subs, vals)
        c.model_init(4, 2001)
        c.sample("stratified", 500, 3000, 77)
        gs, _, _, ga = c.sample_export(1, 0, 3000)
        c.loss_grad("poisson")
        out.append((gs, ga, [c.grad_get(k) for k in range(3)]))
        c.close()
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert out[0][1].max() > 1   # rejections exercised
    for k in range(3):
        assert np.allclose(out[0][2][k], out[1][2][k], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("prec,R", [("fp32", 3), ("fp32", 7), ("fp32", 13), ("fp32", 32), ("fp32", 50),
                                    ("fp32", 128), ("fp64", 2), ("fp64", 8), ("fp64", 24), ("fp64", 64)])
def test_gradient_parity_row_geometries(gcp, orc, prec, R):
    """Every lane geometry of K2 (GL lanes x NV 16-B vectors per row: 1x1 ...
    8x4) against the oracle, up to the largest R the ABI accepts."""
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals, prec=prec, R=R)
    t = orc.Tensor(dims, subs, vals)
    c.sample("stratified", 600, 600, 3001)
    A = _model(c, 3)
    c.loss_grad("poisson")
    G = [c.grad_get(k) for k in range(3)]
    Go, S, _ = orc.sampled_grad(t, A, "poisson", 3001, 0, 0, 600, 600)
    _grad_check(G, Go, S, TOL[prec], f"R={R}/{prec}")
    est = c.loss_estimate("poisson", 1500, 1500, 4001)
    oe, scale = orc.loss_estimate(t, A, "poisson", 4001, 0, 1500, 1500)
    assert abs(est - oe) <= TOL[prec] * scale, (est, oe, abs(est - oe) / scale)


@pytest.mark.parametrize("dims", [(60, 70), (9, 10, 11, 12), (4, 5, 6, 5, 4, 6)])
def test_gradient_parity_orders(gcp, orc, dims):
    """Tensor orders d = 2, 4, 6 (d = 3 and 5 above): ingest order, sample
    indices and the gradient."""
    subs, vals = gcp_synth.chi_kolda(dims, 1500, 3, 1007, loss="gaussian")
    subs, vals = subs.numpy(), vals.numpy() - 1.0
    c = _ctx(gcp, dims, subs, vals, prec="fp64", R=5)
    t = orc.Tensor(dims, subs, vals)
    ss, sv = t.sorted()
    gs, gv = c.tensor_export_sorted(0, len(vals))
    assert np.array_equal(gs, ss) and np.array_equal(gv, sv)
    c.sample("stratified", 500, 700, 3001)
    for stratum, n in ((0, 500), (1, 700)):
        g_s, g_j, _, g_a = c.sample_export(stratum, 0, n)
        o_s, o_j, _, o_a = orc.sample_export(t, stratum, 3001, 0, 0, n, 0, n)
        assert np.array_equal(g_s, o_s) and np.array_equal(g_j, o_j) and np.array_equal(g_a, o_a)
    A = _model(c, len(dims))
    c.loss_grad("gaussian")
    G = [c.grad_get(k) for k in range(len(dims))]
    Go, S, _ = orc.sampled_grad(t, A, "gaussian", 3001, 0, 0, 500, 700)
    _grad_check(G, Go, S, TOL["fp64"], f"d={len(dims)}")


def test_slot_order_survives_model_reinit(gcp, orc, monkeypatch):
    """Regression (round-1 advisor, high): with the slot order on, a model
    re-initialised at another R (another K2 geometry and partial count) keeps
    valid order buffers: the gradient after model_init(16) -> loss_grad ->
    model_init(4) -> loss_grad still matches the oracle."""
    monkeypatch.setenv("GCP_SLOT_ORDER", "1")
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = gcp.Context(0, None, "fp32")
    c.tensor_create(dims, subs, vals)
    t = orc.Tensor(dims, subs, vals)
    for R in (16, 4, 16, 2):
        c.model_init(R, 2001)
        assert c.layout()["slot_order"]
        c.sample("stratified", 1500, 1700, 3001)
        A = _model(c, 3)
        c.loss_grad("poisson")
        G = [c.grad_get(k) for k in range(3)]
        Go, S, _ = orc.sampled_grad(t, A, "poisson", 3001, 0, 0, 1500, 1700)
        _grad_check(G, Go, S, TOL["fp32"], f"reinit R={R}")
    # a replaced tensor rebuilds the per-tensor bucket table
    subs2, vals2 = gcp_synth.chi_kolda(dims, 1800, 4, 1009, loss="poisson")
    subs2, vals2 = subs2.numpy(), vals2.numpy()
    c.tensor_create(dims, subs2, vals2)
    c.model_init(4, 2001)
    t2 = orc.Tensor(dims, subs2, vals2)
    c.sample("stratified", 900, 1100, 3001)
    A = _model(c, 3)
    c.loss_grad("poisson")
    Go, S, _ = orc.sampled_grad(t2, A, "poisson", 3001, 0, 0, 900, 1100)
    _grad_check([c.grad_get(k) for k in range(3)], Go, S, TOL["fp32"], "replaced tensor")


def test_dims_product_overflow_is_an_error(gcp):
    """prod I_k must fit in 128 bits: five modes of 2^32 - 1 do not."""
    c = gcp.Context(0, None, "fp32")
    with pytest.raises(gcp.GcpError) as e:
        c.tensor_create((2 ** 32 - 1,) * 5, np.array([[0, 0, 0, 0, 0]]), np.array([1.0]))
    assert e.value.name == "GCP_E_ARG"
    c.tensor_create((2 ** 32 - 1,) * 4, np.array([[0, 0, 0, 0]]), np.array([1.0]))   # 128 bits: fine


def test_nonzero_index_beyond_2_32(gcp, orc):
    """Reading R11 index map j = floor(W0 N / 2^64) on the device draw path for
    N >= 2^32 (c5 holds 4.69e9 nonzeros; the kernel keeps 32 bits of j in flight
    and re-derives the full j): bit-exact against Philox + Python integers."""
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = _ctx(gcp, dims, subs, vals)
    seed = (11 << 32) | 3005
    for N, rank, it in ((4_687_474_081, 0, 7), (2 ** 32, 3, 0), (2 ** 40 + 12345, 1, 123456), (2 ** 32 - 1, 0, 2)):
        first, count = 1_000_000, 4096
        j = c.debug_nonzero_j(seed, rank, it, N, first, count)
        for s in range(first, first + count, 37):
            o = orc.philox([s, rank, 0, it], [seed & 0xFFFFFFFF, seed >> 32])
            W0 = o[0] | (o[1] << 32)
            assert j[s - first] == (W0 * N) >> 64, (N, s)
        assert j.max() >= 2 ** 32 or N <= 2 ** 32


@pytest.mark.parametrize("membership", ["hash", "sorted"])
def test_lean_ingest_same_tensor(gcp, orc, membership, monkeypatch):
    """The lean ingest (sort of (key, value) pairs, records decoded from the
    sorted keys, hash built from the records -- the path a 4.69e9-nonzero c5
    block takes on one GPU) gives the standard path's tensor: canonical records,
    membership answers and sample draws; and on c1 the oracle's gradient."""
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    t = orc.Tensor(dims, subs, vals)
    monkeypatch.setenv("GCP_INGEST", "lean")
    c = gcp.Context(0, None, "fp32")
    c.set_membership(membership)
    c.tensor_create(dims, subs, vals)
    ss, sv = t.sorted()
    gs, gv = c.tensor_export_sorted(0, len(vals))
    assert np.array_equal(gs, ss) and np.array_equal(gv, sv.astype(np.float32).astype(np.float64))
    rng = np.random.default_rng(3)
    cand = np.stack([rng.integers(0, I, 20000) for I in dims], 1)
    assert np.array_equal(c.tensor_contains(cand), np.array([t.contains(x) for x in cand]))
    c.model_init(4, 2001)
    c.sample("stratified", 1000, 1000, 3001)
    for stratum in (0, 1):
        g_s, g_j, _, g_a = c.sample_export(stratum, 0, 1000)
        o_s, o_j, _, o_a = orc.sample_export(t, stratum, 3001, 0, 0, 1000, 0, 1000)
        assert np.array_equal(g_s, o_s) and np.array_equal(g_j, o_j) and np.array_equal(g_a, o_a)
    A = _model(c, 3)
    c.loss_grad("poisson")
    Go, S, _ = orc.sampled_grad(t, A, "poisson", 3001, 0, 0, 1000, 1000)
    _grad_check([c.grad_get(k) for k in range(3)], Go, S, TOL["fp32"], f"lean/{membership}")
    # a c4-shaped block of 2e6 nonzeros: lean and standard ingest agree record for record
    d4 = gcp_synth.CONFIGS["c4"]["dims"]
    s4, v4 = gcp_synth.chi_kolda(d4, 2_000_000, 16, 1004, loss="gaussian", device="cuda")
    s4, v4 = s4.cpu().numpy(), v4.cpu().numpy()
    out = []
    cand = np.stack([rng.integers(0, I, 50000) for I in d4], 1)
    cand[:20000] = s4[:20000]
    for mode in ("lean", "standard"):
        monkeypatch.setenv("GCP_INGEST", mode)
        cx = gcp.Context(0, None, "fp32")
        cx.set_membership(membership)
        cx.tensor_create(d4, s4, v4)
        out.append((cx.tensor_export_sorted(0, len(v4)), cx.tensor_contains(cand)))
        cx.close()
    assert np.array_equal(out[0][0][0], out[1][0][0]) and np.array_equal(out[0][0][1], out[1][0][1])
    assert np.array_equal(out[0][1], out[1][1]) and out[0][1][:20000].all()


def test_device_philox_kat_and_curand(gcp):
    """the sampler's device Philox4x32-10 reproduces the Random123
    known-answer vectors (tests/golden) and equals curand's
    curand_Philox4x32_10 on 1e5 random (counter, key) pairs."""
    from conftest import GOLDEN
    dims = (20, 30, 40)
    subs, vals = _tensor("poisson")
    c = gcp.Context(0, None, "fp32")
    c.tensor_create(dims, subs, vals)
    kat = []
    for line in (GOLDEN / "philox4x32_10_kat.txt").read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            kat.append([int(x, 16) for x in line.split()])
    kat = np.array(kat, dtype=np.uint64).astype(np.uint32)
    ours, cur = c.debug_philox(kat[:, :6])
    assert np.array_equal(ours, kat[:, 6:10]) and np.array_equal(cur, kat[:, 6:10])
    rng = np.random.default_rng(11)
    x = rng.integers(0, 2 ** 32, size=(100_000, 6), dtype=np.uint64).astype(np.uint32)
    ours, cur = c.debug_philox(x)
    assert np.array_equal(ours, cur)
