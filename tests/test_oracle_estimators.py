"""Pins for the oracle's sampled estimators, Adam, grid and multi-rank loops."""
import math

import numpy as np
import pytest
from conftest import read_golden

import gcp_synth

LOSSES = ["gaussian", "poisson", "bernoulli"]


def _fixture(loss, dims=(5, 4, 3), nnz=12, R=3, seed=0):
    rng = np.random.default_rng(seed)
    vals = {"gaussian": "normal", "poisson": "counts", "bernoulli": "ones"}[loss]
    subs, v = gcp_synth.uniform_sparse(dims, nnz, seed=seed + 1, values=vals)
    lo = 0.2 if loss != "bernoulli" else -1.0
    A = [rng.uniform(lo, 1.0, size=(I, R)) for I in dims]
    return dims, subs, v, A


@pytest.mark.parametrize("strategy", ["stratified", "semi"])
@pytest.mark.parametrize("loss", LOSSES)
def test_fused_equals_nonfused_bitwise(orc, loss, strategy):
    """Fused Sampling-MTTKRP is the non-fused Y~ -> MTTKRP pipeline
    with the same entries in the same order."""
    dims, subs, v, A = _fixture(loss, seed=3)
    t = orc.Tensor(dims, subs, v)
    for it in range(3):
        G, _, _ = orc.sampled_grad(t, A, loss, 99, 0, it, 17, 23, strategy)
        coords, y = orc.build_Y(t, A, loss, 99, 0, it, 17, 23, strategy)
        G2 = orc.mttkrp(t, A, coords, y)
        for a, b in zip(G, G2):
            assert np.array_equal(a, b)


def test_duplicate_samples_carry_equal_values(orc):
    """P:548-552 footnote: repeated entries of Y~ have the same value."""
    dims, subs, v, A = _fixture("poisson", dims=(3, 3, 2), nnz=5, seed=4)
    t = orc.Tensor(dims, subs, v)
    coords, y = orc.build_Y(t, A, "poisson", 5, 0, 0, 40, 40)
    seen = {}
    for c, val in zip(map(tuple, coords), y):
        seen.setdefault(c, set()).add(val)
    assert any(len(c) for c in seen)
    assert max(len(s) for s in seen.values()) == 1
    assert len(seen) < 80  # duplicates did occur


def _mean_grad(orc, t, A, loss, strategy, K, p, q, seed0=1000):
    acc = [np.zeros_like(a) for a in A]
    sq = [np.zeros_like(a) for a in A]
    for s in range(K):
        G, _, _ = orc.sampled_grad(t, A, loss, seed0 + s, 0, 0, p, q, strategy, with_scale=False)
        for k in range(len(A)):
            acc[k] += G[k]
            sq[k] += G[k] ** 2
    mean = [a / K for a in acc]
    se = [np.sqrt(np.maximum(s / K - m ** 2, 0) / K) for s, m in zip(sq, mean)]
    return mean, se


@pytest.mark.parametrize("loss", LOSSES)
def test_stratified_gradient_unbiased(orc, loss):
    """E[G~] = exact dense gradient (P:525-537 weights N/p, (M-N)/q).
    SPEC S:211: 5x4x3, R=3, 10,000 draws, < 2% per mode; plus a 3-SE gate."""
    dims, subs, v, A = _fixture(loss, seed=5)
    t = orc.Tensor(dims, subs, v)
    exact = orc.full_grad(t, A, loss)
    mean, se = _mean_grad(orc, t, A, loss, "stratified", 10000, 10, 10)
    for k in range(3):
        err = np.linalg.norm(mean[k] - exact[k])
        assert err < 3 * np.linalg.norm(se[k]) + 1e-12
        if loss == "poisson":  # SPEC's fixed fixture is Poisson
            assert err / np.linalg.norm(exact[k]) < 0.02


@pytest.mark.parametrize("loss", LOSSES)
def test_semi_stratified_expectation(orc, loss):
    """Reading R6: with zero weight (M-N)/q and nonzero values w(f'(x,m)-f'(0,m)),
    E[G~] = full_grad(X) - (N/M) * full_grad(empty tensor)."""
    dims, subs, v, A = _fixture(loss, seed=6)
    t = orc.Tensor(dims, subs, v)
    t0 = orc.Tensor(dims, np.zeros((0, 3), np.int64), np.zeros(0))
    N, M = len(v), math.prod(dims)
    gx, g0 = orc.full_grad(t, A, loss), orc.full_grad(t0, A, loss)
    expect = [a - N / M * b for a, b in zip(gx, g0)]
    mean, se = _mean_grad(orc, t, A, loss, "semi", 10000, 10, 10, seed0=5000)
    for k in range(3):
        err = np.linalg.norm(mean[k] - expect[k])
        assert err < 3 * np.linalg.norm(se[k]) + 1e-12


@pytest.mark.parametrize("loss", LOSSES)
def test_loss_estimate_unbiased(orc, loss):
    dims, subs, v, A = _fixture(loss, seed=7)
    t = orc.Tensor(dims, subs, v)
    F = orc.full_loss(t, A, loss)
    ests = np.array([orc.loss_estimate(t, A, loss, 7000 + s, 0, 10, 10)[0] for s in range(10000)])
    assert abs(ests.mean() - F) < 3 * ests.std() / 100 + 1e-12
    if loss == "poisson":
        assert abs(ests.mean() - F) / abs(F) < 0.02


def test_loss_estimate_exact_at_optimum(orc):
    """Gaussian model equal to the data -> every term is zero."""
    dims = (4, 3, 2)
    A = [np.array([[1.0], [2.0], [0.5], [1.5]]), np.array([[1.0], [3.0], [2.0]]), np.array([[2.0], [1.0]])]
    M = np.einsum("ir,jr,kr->ijk", *A)
    subs = np.array(np.nonzero(M)).T
    # every entry is nonzero in M, so make a sparse X by zeroing one factor row
    A[0][2] = 0.0
    M = np.einsum("ir,jr,kr->ijk", *A)
    subs = np.array(np.nonzero(M)).T
    t = orc.Tensor(dims, subs, M[tuple(subs.T)])
    est, _ = orc.loss_estimate(t, A, "gaussian", 3, 0, 50, 50)
    assert est == 0.0
    G, _, _ = orc.sampled_grad(t, A, "gaussian", 3, 0, 0, 30, 30)
    assert all((g == 0).all() for g in G)


def test_adam_worked_example_and_invariants(orc):
    g = {r[0]: r for r in read_golden("worked_examples.txt")}
    A, G, B, Cm = (np.array([1.0]), np.array([1.0]), np.zeros(1), np.zeros(1))
    orc.adam(A, G, B, Cm, 1, 1e-3, 0.9, 0.999, 1e-8)
    assert A[0] == pytest.approx(float(g["adam_first_step"][2]), abs=1e-15)
    # Constant gradient g: bias correction makes B^ = g, C^ = g^2 at every t, so
    # every step moves exactly alpha*g/sqrt(g^2+eps) (for any beta; Table 3 values).
    for beta1, beta2 in [(0.630219, 0.966996), (0.603286, 0.991181), (0.9, 0.999)]:
        rng = np.random.default_rng(1)
        gv = rng.normal(size=50)
        A = rng.normal(size=50)
        B, Cm = np.zeros(50), np.zeros(50)
        for t in range(1, 101):
            A0 = A.copy()
            orc.adam(A, gv.copy(), B, Cm, t, 0.035817, beta1, beta2, 1.388768e-13)
            step = 0.035817 * gv / np.sqrt(gv ** 2 + 1.388768e-13)
            assert np.allclose(A0 - A, step, rtol=1e-9, atol=1e-15)
    # zero gradient from zero moments is a fixed point; clamp keeps A >= l
    A = np.array([0.3, -0.2, 0.0])
    orc.adam(A, np.zeros(3), np.zeros(3), np.zeros(3), 1, 1e-3)
    assert np.array_equal(A, [0.3, -0.2, 0.0])
    A = np.array([0.0005, 0.5, 0.00001])
    orc.adam(A, np.ones(3), np.zeros(3), np.zeros(3), 1, 1e-3, lower=0.0)
    assert (A >= 0).all() and A[0] == 0.0 and A[2] == 0.0
    # NaN propagates through the clamp (comparison form, reading R9)
    A = np.array([0.5])
    orc.adam(A, np.array([np.nan]), np.zeros(1), np.zeros(1), 1, 1e-3, lower=0.0)
    assert np.isnan(A[0])


def test_adam_single_array_equals_per_mode(orc):
    """one pass over the contiguous array == per-mode updates."""
    rng = np.random.default_rng(3)
    sizes = [12, 7, 20]
    A, G = rng.normal(size=39), rng.normal(size=39)
    B, Cm = rng.normal(size=39) * 0.1, rng.uniform(size=39) * 0.1
    A2, B2, C2 = A.copy(), B.copy(), Cm.copy()
    orc.adam(A, G, B, Cm, 5, 1e-2, 0.9, 0.999, 1e-8)
    off = 0
    for n in sizes:
        a, b, c = A2[off:off + n].copy(), B2[off:off + n].copy(), C2[off:off + n].copy()
        orc.adam(a, G[off:off + n].copy(), b, c, 5, 1e-2, 0.9, 0.999, 1e-8)
        assert np.array_equal(a, A[off:off + n]) and np.array_equal(b, B[off:off + n])
        off += n


def test_grid_plans_pinned_and_bruteforce(orc):
    for dims_s, P, grid_s, obj in read_golden("grid_plans.txt"):
        dims = [int(x) for x in dims_s.split("x")]
        grid, o = orc.grid_plan(int(P), dims)
        assert grid == tuple(int(x) for x in grid_s.split(","))
        assert o == float(obj)
    # independent brute force (itertools) over small P and Table 1's synthetic shape
    import itertools
    dims = (300, 200, 100)
    for P in range(1, 65):
        best = None
        for tup in itertools.product(range(1, P + 1), repeat=3):
            if math.prod(tup) != P:
                continue
            val = sum(I * P // n for I, n in zip(dims, tup))
            if best is None or val < best[0] or (val == best[0] and tup < best[1]):
                best = (val, tup)
        grid, o = orc.grid_plan(P, dims)
        assert (o, grid) == (best[0], best[1])
    # P prime with a unique largest mode -> all of P on that mode
    assert orc.grid_plan(7, (10, 50, 20))[0] == (1, 7, 1)


def test_alloc_and_blocks(orc):
    g = {r[0]: r for r in read_golden("worked_examples.txt")}
    assert [orc.alloc_count(10, 4, w) for w in range(4)] == [int(x) for x in g["alloc_p10_P4"][2].split(",")]
    dims = (10, 7, 5)
    grid = (2, 3, 1)
    cover = np.zeros(dims, int)
    for w in range(6):
        lo, hi = orc.block_bounds(dims, grid, w)
        cover[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] += 1
    assert (cover == 1).all()
    assert orc.rank_coords(5, grid) == (1, 2, 0)


def test_multirank_gradient_unbiased_and_P1_identity(orc):
    dims, subs, v, A = _fixture("poisson", dims=(6, 5, 4), nnz=30, seed=9)
    t = orc.Tensor(dims, subs, v)
    blocks, grid = orc.split_blocks(dims, subs, v, 1)
    G1, _, _ = orc.sync_gradient(blocks, A, "poisson", 11, 2, 40, 40)
    G, _, _ = orc.sampled_grad(t, A, "poisson", 11, 0, 2, 40, 40)
    assert all(np.array_equal(a, b) for a, b in zip(G1, G))
    # P = 4 ranks, local weights (reading R13): sum over ranks is unbiased
    blocks, grid = orc.split_blocks(dims, subs, v, 4)
    assert math.prod(grid) == 4
    exact = orc.full_grad(t, A, "poisson")
    K = 3000
    acc = [np.zeros_like(a) for a in A]
    sq = [np.zeros_like(a) for a in A]
    for s in range(K):
        Gs, _, _ = orc.sync_gradient(blocks, A, "poisson", 100 + s, 0, 16, 16)
        for k in range(3):
            acc[k] += Gs[k]
            sq[k] += Gs[k] ** 2
    for k in range(3):
        m = acc[k] / K
        se = np.sqrt(np.maximum(sq[k] / K - m ** 2, 0) / K)
        assert np.linalg.norm(m - exact[k]) < 3 * np.linalg.norm(se)


def test_fit_collapses_and_annealing(orc):
    dims, subs, v, _ = _fixture("poisson", dims=(8, 6, 5), nnz=40, seed=12)
    A0 = orc.factor_init(7, dims, 3)
    blocks, grid = orc.split_blocks(dims, subs, v, 1)
    kw = dict(epochs=3, iters=5, s_nz=20, s_z=20, f_nz=50, f_z=50, seed=1, fseed=2, rate=1e-2)
    As, hs, _ = orc.fit(blocks, grid, A0, "poisson", mode="sync", **kw)
    # P = 1: LocalSGD averaging is the identity; FedAdam with tau beyond the run never syncs
    Aa, ha, _ = orc.fit(blocks, grid, A0, "poisson", mode="async", tau=2, **kw)
    Af, hf, _ = orc.fit(blocks, grid, A0, "poisson", mode="fedadam", tau=1000, **kw)
    for k in range(3):
        assert np.array_equal(As[k], Aa[0][k]) and np.array_equal(As[k], Af[0][k])
    assert hs == ha == hf
    # accepted losses strictly decrease; rate non-increasing
    acc = [h[0] for h in hs if h[2]]
    assert all(a > b for a, b in zip(acc, acc[1:]))
    # forced failure: rate 0 -> no progress -> exactly max_fails rejected epochs
    A1, h1, _ = orc.fit(blocks, grid, A0, "poisson", mode="sync", **{**kw, "rate": 0.0, "epochs": 10})
    assert len(h1) == 3 and not any(h[2] for h in h1)
    assert all(np.array_equal(a, b) for a, b in zip(A1, A0))


def test_async_replicas_identical_after_sync(orc):
    dims, subs, v, _ = _fixture("poisson", dims=(8, 6, 5), nnz=40, seed=13)
    A0 = orc.factor_init(8, dims, 2)
    blocks, grid = orc.split_blocks(dims, subs, v, 4, grid=(1, 2, 2))
    kw = dict(epochs=1, iters=4, s_nz=20, s_z=20, f_nz=20, f_z=20, seed=3, fseed=4, rate=1e-2)
    # tau = 4: the last iteration starts with an averaging step; the models differ
    # afterwards only by that iteration's local step.  With rate 0 they are equal.
    Aw, _, _ = orc.fit(blocks, grid, A0, "poisson", mode="async", tau=4, **{**kw, "rate": 0.0})
    for k in range(3):
        for grp in orc.slice_groups(grid, k):
            lo, hi = blocks[grp[0]].lo[k], blocks[grp[0]].hi[k]
            for w in grp[1:]:
                assert np.array_equal(Aw[w][k][lo:hi], Aw[grp[0]][k][lo:hi])


@pytest.mark.parametrize("nthreads", [1, 3, 8])
def test_openmp_timing_variant_matches_serial(orc, nthreads):
    """The OpenMP variant timed as the CPU baseline
    computes the serial oracle's estimator: same draws, sums reordered only."""
    dims, subs, v, A = _fixture("poisson", dims=(9, 8, 7), nnz=60, seed=31)
    t = orc.Tensor(dims, subs, v)
    G, _, ls = orc.sampled_grad(t, A, "poisson", 5, 0, 3, 301, 457, with_scale=False)
    Gp, lp = orc.sampled_grad_par(t, A, "poisson", 5, 0, 3, 301, 457, nthreads=nthreads)
    for a, b in zip(G, Gp):
        assert np.allclose(a, b, rtol=1e-12, atol=1e-12 * np.abs(a).max())
    assert lp == pytest.approx(ls, rel=1e-12)
    e, _ = orc.loss_estimate(t, A, "poisson", 9, 0, 200, 300)
    assert orc.loss_estimate_par(t, A, "poisson", 9, 0, 200, 300, nthreads=nthreads) == pytest.approx(e, rel=1e-12)
    flat = np.concatenate([a.ravel() for a in A])
    g = np.concatenate([a.ravel() for a in G])
    a1, b1, c1 = flat.copy(), np.zeros_like(flat), np.zeros_like(flat)
    a2, b2, c2 = flat.copy(), np.zeros_like(flat), np.zeros_like(flat)
    orc.adam(a1, g, b1, c1, 1, 1e-2, lower=0.0)
    orc.adam_par(a2, g, b2, c2, 1, 1e-2, lower=0.0, nthreads=nthreads)
    assert np.array_equal(a1, a2) and np.array_equal(b1, b2) and np.array_equal(c1, c2)
