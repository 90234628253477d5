"""Pins for the oracle's model value, losses, MTTKRP and exact gradient.

Each check compares the oracle with something other than itself: worked
examples (tests/golden/worked_examples.txt), dense unfolding x explicitly
formed Khatri-Rao products, central finite differences, and closed forms
(the CP least-squares gradient, the Poisson gradient split)."""
import math

import numpy as np
import pytest
from conftest import read_golden

import gcp_synth

LOSSES = ["gaussian", "poisson", "bernoulli"]


def _golden():
    return {r[0]: r for r in read_golden("worked_examples.txt")}


def test_model_value_worked_examples(orc):
    g = _golden()
    t = orc.Tensor((2, 2, 2), np.zeros((0, 3), np.int64), np.zeros(0))
    A = [np.ones((2, 2))] * 3
    assert orc.model_value(t, A, (1, 0, 1)) == float(g["model_all_ones"][2])
    A = [np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]]), np.array([[5.0], [6.0]])]
    assert orc.model_value(t, A, (1, 0, 1)) == float(g["model_rank1"][2])
    rng = np.random.default_rng(0)
    A = [rng.uniform(size=(2, 3)) for _ in range(3)]
    A[0][1] = 0.0
    assert orc.model_value(t, A, (1, 1, 0)) == float(g["model_zero_row"][2])
    # lambda enters multiplicatively per component
    A = [rng.uniform(size=(2, 3)) for _ in range(3)]
    lam = np.array([2.0, -1.0, 0.5])
    want = sum(lam[r] * A[0][0, r] * A[1][1, r] * A[2][1, r] for r in range(3))
    assert abs(orc.model_value(t, A, (0, 1, 1), lam) - want) < 1e-15


def test_loss_worked_examples(orc):
    g = _golden()
    assert orc.loss_f("gaussian", 2.5, 2.5) == 0.0
    assert orc.loss_f("gaussian", 1, 3) == float(g["gauss_f"][2])
    assert orc.loss_f("poisson", 0, 3) == float(g["poisson_f_zero"][2])
    assert abs(orc.loss_df("poisson", 2, 1) - float(g["poisson_df"][2])) < 1e-9
    assert orc.loss_df("gaussian", 4, 4) == 0.0
    assert abs(orc.loss_f("bernoulli", 0, 0) - math.log(2)) < 1e-16
    assert orc.loss_df("bernoulli", 0, 0) == 0.5
    assert orc.loss_df("bernoulli", 1, 0) == -0.5
    assert orc.loss_lower("poisson") == 0.0
    assert orc.loss_lower("gaussian") == -math.inf


@pytest.mark.parametrize("loss", LOSSES)
def test_loss_derivative_finite_difference(orc, loss):
    rng = np.random.default_rng(1)
    for _ in range(20):
        if loss == "bernoulli":
            x, m = float(rng.integers(0, 2)), rng.uniform(-6, 6)
        else:
            x, m = rng.uniform(0, 5), rng.uniform(0.2, 5)
        h = 1e-5
        fd = (orc.loss_f(loss, x, m + h) - orc.loss_f(loss, x, m - h)) / (2 * h)
        assert abs(orc.loss_df(loss, x, m) - fd) <= 1e-6 * max(1.0, abs(fd))


def test_bernoulli_stable_at_large_margin(orc):
    assert orc.loss_f("bernoulli", 0, 800.0) == pytest.approx(800.0)
    assert orc.loss_f("bernoulli", 1, -800.0) == pytest.approx(800.0)
    assert orc.loss_df("bernoulli", 0, -800.0) == pytest.approx(0.0, abs=1e-300)
    assert orc.loss_df("bernoulli", 0, 800.0) == 1.0
    # matches the naive formula where it does not overflow
    for m in (-3.0, -0.1, 0.7, 5.0):
        assert orc.loss_f("bernoulli", 1, m) == pytest.approx(math.log1p(math.exp(m)) - m, rel=1e-14)


def _khatri_rao(mats):
    """Column-wise Kronecker product, first matrix slowest (C order)."""
    out = mats[0]
    for B in mats[1:]:
        out = (out[:, None, :] * B[None, :, :]).reshape(-1, out.shape[1])
    return out


def _dense_mttkrp(Y, A, k, lam):
    """Brute force: unfold Y in mode k (C order over the remaining modes) times
    the explicitly formed Khatri-Rao product of the other factors, times diag(lam)."""
    d = Y.ndim
    Yk = np.moveaxis(Y, k, 0).reshape(Y.shape[k], -1)
    Z = _khatri_rao([A[j] for j in range(d) if j != k])
    return Yk @ Z * lam[None, :]


@pytest.mark.parametrize("dims", [(4, 3, 2), (3, 3, 3, 2)])
def test_sparse_mttkrp_equals_dense_khatri_rao(orc, dims):
    rng = np.random.default_rng(2)
    R = 2 if len(dims) == 3 else 3
    nnz = int(np.prod(dims)) // 2
    subs, vals = gcp_synth.uniform_sparse(dims, nnz, seed=3)
    t = orc.Tensor(dims, subs, vals)
    A = [rng.normal(size=(I, R)) for I in dims]
    lam = rng.uniform(0.5, 2, size=R)
    # an entry list with duplicates (as Y~ may have)
    coords = np.concatenate([subs, subs[:5]])
    y = rng.normal(size=len(coords))
    G = orc.mttkrp(t, A, coords, y, lam)
    Y = np.zeros(dims)
    np.add.at(Y, tuple(coords.T), y)
    for k in range(len(dims)):
        ref = _dense_mttkrp(Y, A, k, lam)
        assert np.allclose(G[k], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def _dense(dims, subs, vals):
    X = np.zeros(dims)
    X[tuple(subs.T)] = vals
    return X


@pytest.mark.parametrize("loss", LOSSES)
def test_full_gradient_finite_differences(orc, loss):
    dims = (3, 3, 3)
    R = 2
    rng = np.random.default_rng(4)
    if loss == "bernoulli":
        subs, vals = gcp_synth.uniform_sparse(dims, 9, seed=5, values="ones")
        A = [rng.normal(scale=0.8, size=(3, R)) for _ in dims]
    else:
        subs, vals = gcp_synth.uniform_sparse(dims, 9, seed=5, values="counts")
        A = [rng.uniform(0.3, 1.2, size=(3, R)) for _ in dims]
    lam = np.array([1.0, 0.7])
    t = orc.Tensor(dims, subs, vals)
    G = orc.full_grad(t, A, loss, lam)
    h = 1e-6
    for k in range(3):
        for i in range(3):
            for r in range(R):
                Ap = [a.copy() for a in A]
                Am = [a.copy() for a in A]
                Ap[k][i, r] += h
                Am[k][i, r] -= h
                fd = (orc.full_loss(t, Ap, loss, lam) - orc.full_loss(t, Am, loss, lam)) / (2 * h)
                assert abs(G[k][i, r] - fd) <= 1e-5 * max(1.0, abs(fd))


def test_gaussian_gradient_is_cp_least_squares_gradient(orc):
    """Full GCP-Gaussian gradient = 2[A^(k) L (*_{j!=k} A^(j)T A^(j)) L - X_(k) Z_k L]
    (the CP least-squares gradient; second term is the MTTKRP of X alone)."""
    dims = (5, 4, 6)
    R = 3
    rng = np.random.default_rng(6)
    subs, vals = gcp_synth.uniform_sparse(dims, 40, seed=7, values="normal")
    t = orc.Tensor(dims, subs, vals)
    A = [rng.normal(size=(I, R)) for I in dims]
    lam = rng.uniform(0.5, 1.5, size=R)
    L = np.diag(lam)
    X = _dense(dims, subs, vals)
    G = orc.full_grad(t, A, "gaussian", lam)
    for k in range(3):
        H = np.ones((R, R))
        for j in range(3):
            if j != k:
                H *= A[j].T @ A[j]
        mttkrp_X = np.einsum("ijk,jr,kr->ir", np.moveaxis(X, k, 0),
                             *[A[j] for j in range(3) if j != k]) * lam
        ref = 2 * (A[k] @ L @ H @ L - mttkrp_X)
        assert np.allclose(G[k], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_poisson_gradient_closed_form(orc):
    """Poisson f'(0,m) = 1, so G^(k)[i,r] = lam_r prod_{j!=k} colsum_r(A^(j))
    - sum_{nz with i_k = i} x/(m+eps) lam_r prod_{j!=k} a."""
    dims = (6, 5, 4)
    R = 3
    rng = np.random.default_rng(8)
    subs, vals = gcp_synth.uniform_sparse(dims, 30, seed=9, values="counts")
    t = orc.Tensor(dims, subs, vals)
    A = [rng.uniform(0.1, 1, size=(I, R)) for I in dims]
    lam = rng.uniform(0.5, 1.5, size=R)
    G = orc.full_grad(t, A, "poisson", lam)
    for k in range(3):
        ref = np.zeros((dims[k], R))
        cs = np.ones(R) * lam
        for j in range(3):
            if j != k:
                cs = cs * A[j].sum(axis=0)
        ref[:] = cs
        for c, x in zip(subs, vals):
            m = sum(lam[r] * A[0][c[0], r] * A[1][c[1], r] * A[2][c[2], r] for r in range(R))
            z = lam.copy()
            for j in range(3):
                if j != k:
                    z = z * A[j][c[j]]
            ref[c[k]] -= x / (m + 1e-10) * z
        assert np.allclose(G[k], ref, rtol=1e-12, atol=1e-13)


def test_poisson_exact_grad_at_scale_matches_enumeration(orc):
    """oracle.poisson_exact_grad (the O(N d R) closed form used as the exact
    target at c2 scale) equals the enumerated gradient of F."""
    for dims, R, nnz, seed in (((6, 5, 4), 3, 30, 19), ((7, 3, 5, 4), 2, 50, 20)):
        rng = np.random.default_rng(seed)
        subs, vals = gcp_synth.uniform_sparse(dims, nnz, seed=seed + 1, values="counts")
        t = orc.Tensor(dims, subs, vals)
        A = [rng.uniform(0.1, 1, size=(I, R)) for I in dims]
        lam = rng.uniform(0.5, 1.5, size=R)
        G = orc.full_grad(t, A, "poisson", lam)
        Gs = orc.poisson_exact_grad(subs, vals, A, lam, chunk=7)   # ragged chunks
        for k in range(len(dims)):
            assert np.allclose(Gs[k], G[k], rtol=1e-12, atol=1e-12 * np.abs(G[k]).max())


def test_full_loss_closed_forms(orc):
    dims = (5, 4, 3)
    R = 2
    rng = np.random.default_rng(10)
    subs, vals = gcp_synth.uniform_sparse(dims, 20, seed=11, values="counts")
    t = orc.Tensor(dims, subs, vals)
    A = [rng.uniform(0.1, 1, size=(I, R)) for I in dims]
    lam = np.array([1.3, 0.6])
    M = np.einsum("r,ir,jr,kr->ijk", lam, *A)
    X = _dense(dims, subs, vals)
    # Gaussian: ||X||^2 - 2<X, M> + lam^T (*_k A^(k)T A^(k)) lam
    H = np.ones((R, R))
    for a in A:
        H *= a.T @ a
    gauss = (X ** 2).sum() - 2 * (X * M).sum() + lam @ H @ lam
    assert orc.full_loss(t, A, "gaussian", lam) == pytest.approx(gauss, rel=1e-12)
    # Poisson: sum_r lam_r prod_k colsum_r(A^(k)) - sum_nz x log(m + eps)
    pois = (lam * np.prod([a.sum(0) for a in A], axis=0)).sum() - \
        sum(x * math.log(M[tuple(c)] + 1e-10) for c, x in zip(subs, vals))
    assert orc.full_loss(t, A, "poisson", lam) == pytest.approx(pois, rel=1e-12)
    # all-zero 2x2x2, rank-1 all-ones, Poisson -> 8
    t0 = orc.Tensor((2, 2, 2), np.zeros((0, 3), np.int64), np.zeros(0))
    assert orc.full_loss(t0, [np.ones((2, 1))] * 3, "poisson") == pytest.approx(8.0, rel=1e-12)
