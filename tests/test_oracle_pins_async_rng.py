"""Pins that tie the oracle's multi-rank layer and its RNG counter layout to the
paper / the documented readings rather than to the GPU path.

* LocalSGD averaging (Alg. 3, reading R16): after a sync every
  replica equals the arithmetic mean of its slice group's pre-sync replicas
  (divisor g_k, not "numMPIRanks").
* FedAdam (Alg. 4, reading R17): one server step at a tau that
  fires equals a hand-computed Alg. 1 step on U with gradient
  sum_w (U - M_w), followed by M <- U; U moves towards the clients.
* Reading R11: nonzero and zero draws, f-samples and the iteration word are
  recomputed from the KAT-pinned Philox with the documented counter
  (slot, rank, kind<<28 | attempt<<4 | group, it) and key (lo32, hi32 seed),
  and the range map floor(W n / 2^64) written out in Python integers.
"""
import math

import numpy as np
import pytest

import gcp_synth


def _words(orc, seed, slot, rank, kind, attempt, group, it):
    o = orc.philox([slot, rank, (kind << 28) | (attempt << 4) | group, it],
                   [seed & 0xFFFFFFFF, seed >> 32])
    return o[0] | (o[1] << 32), o[2] | (o[3] << 32)


def _rmap(W, n):
    return (W * n) >> 64          # floor(W n / 2^64), exact in Python integers


def _async_setup(orc, mode, tau, seed=13):
    dims = (8, 6, 5)
    subs, v = gcp_synth.uniform_sparse(dims, 40, seed=seed, values="counts")
    A0 = orc.factor_init(8, dims, 2)
    blocks, grid = orc.split_blocks(dims, subs, v, 4, grid=(1, 2, 2))
    run = orc.MultiRank(blocks, grid, A0, "poisson", mode, tau=tau, meta_rate=3e-2)
    return run, blocks, grid


def _snapshot(run):
    return {key: [[a.copy() for a in per_rank] for per_rank in run.st[key]] for key in ("A", "U")}


def test_localsgd_sync_is_slice_group_mean(orc):
    """Alg. 3 lines 2-4: A^(k) block <- (1/g_k) sum over the slice group (R16).
    Grid (1,2,2) at P=4: g_1 = 4 (= P), g_2 = g_3 = 2 (!= P), so both a missing
    division and a division by the rank count fail."""
    run, blocks, grid = _async_setup(orc, "async", tau=4)
    for it in range(3):                       # (it+1) % 4 != 0: local steps only
        run.iteration(it, seed=5, s_nz=20, s_z=20, rate=5e-2)
    pre = _snapshot(run)["A"]
    # replicas really differ before the sync (else the test proves nothing)
    assert any(not np.array_equal(pre[0][k], pre[w][k])
               for k in range(3) for w in range(1, 4) if blocks[w].lo[k] == blocks[0].lo[k])
    run.iteration(3, seed=5, s_nz=20, s_z=20, rate=0.0)   # sync fires, then a rate-0 local step
    for k in range(3):
        groups = orc.slice_groups(grid, k)
        assert sorted(len(g) for g in groups) == ([4] if k == 0 else [2, 2])
        for grp in groups:
            mean = np.stack([pre[w][k] for w in grp]).mean(axis=0)
            for w in grp:
                np.testing.assert_allclose(run.st["A"][w][k], mean, rtol=1e-15, atol=0)


def test_fedadam_server_step_hand_computed(orc):
    """Alg. 4 (body read literally, R17): S = sum_w (U - M_w) over the slice group;
    one Alg. 1 step on U with gradient S from zero server moments (t = 1,
    eps inside the sqrt, clamp at l = 0 for Poisson); M <- U."""
    b1, b2, eps, alpha = 0.9, 0.999, 1e-8, 3e-2
    run, blocks, grid = _async_setup(orc, "fedadam", tau=4)
    for it in range(3):
        run.iteration(it, seed=6, s_nz=20, s_z=20, rate=5e-2)
    snap = _snapshot(run)
    M, U = snap["A"], snap["U"]
    run.iteration(3, seed=6, s_nz=20, s_z=20, rate=0.0)
    moved = 0
    for k in range(3):
        for grp in orc.slice_groups(grid, k):
            u = U[grp[0]][k]
            for w in grp:
                assert np.array_equal(U[w][k], u)       # one server copy per group
            S = sum(u - M[w][k] for w in grp)
            Bs = (1 - b1) * S
            Cs = (1 - b2) * S * S
            expect = u - alpha * (Bs / (1 - b1)) / np.sqrt(Cs / (1 - b2) + eps)
            expect = np.where(expect < 0.0, 0.0, expect)
            for w in grp:
                np.testing.assert_allclose(run.st["A"][w][k], expect, rtol=1e-13, atol=1e-15)
                np.testing.assert_allclose(run.st["U"][w][k], expect, rtol=1e-13, atol=1e-15)
            # direction: the server copy moves towards the clients' mean
            mbar = np.stack([M[w][k] for w in grp]).mean(axis=0)
            big = np.abs(S) > 1e-3
            assert np.all(np.sign(expect - u)[big] == np.sign(mbar - u)[big])
            moved += int(big.sum())
    assert moved > 20
    assert run.st["ts"] == [1, 1, 1, 1]


def _rng_fixture(orc):
    dims = (4, 5, 3, 4, 6)                      # d = 5: Philox groups 0, 1, 2
    subs, v = gcp_synth.uniform_sparse(dims, 300, seed=21, values="counts")   # rho ~ 0.21
    blocks, grid = orc.split_blocks(dims, subs, v, 2)
    return dims, blocks[1], grid                # rank 1: the rank word matters


def test_r11_nonzero_draws_from_documented_counter(orc):
    dims, t, _ = _rng_fixture(orc)
    ss, _ = t.sorted()
    seed, it, rank = (7 << 32) | 12345, 5, 1     # both key words nonzero
    n = 200
    subs, j, _, att = orc.sample_export(t, 0, seed, rank, it, n, 0, n)
    for s in range(n):
        W0, _ = _words(orc, seed, s, rank, 0, 0, 0, it)
        jj = _rmap(W0, t.nnz)
        assert j[s] == jj and tuple(subs[s]) == tuple(ss[jj]) and att[s] == 1
    # f-samples: kind 2 (reading R11), any iteration word passed through
    fs, fj, _, _ = orc.sample_export(t, 0, seed, rank, 0xFFFFFFFF, n, 0, n, f_samples=True)
    for s in range(0, n, 7):
        W0, _ = _words(orc, seed, s, rank, 2, 0, 0, 0xFFFFFFFF)
        assert fj[s] == _rmap(W0, t.nnz)


def test_r11_zero_draws_from_documented_counter(orc):
    dims, t, _ = _rng_fixture(orc)
    seed, it, rank = (3 << 32) | 999, 2, 1
    q = 400
    subs, j, _, att = orc.sample_export(t, 1, seed, rank, it, q, 0, q)
    present = set(map(tuple, t.sorted()[0]))
    retried = 0
    for s in range(q):
        # replay the rejection loop from the documented counter
        for a in range(att[s]):
            c = []
            for k in range(t.d):
                W = _words(orc, seed, s, rank, 1, a, k // 2, it)[k % 2]
                c.append(t.lo[k] + _rmap(W, t.hi[k] - t.lo[k]))
            if a < att[s] - 1:
                assert tuple(c) in present      # rejected attempts were nonzeros
        assert tuple(subs[s]) == tuple(c) and tuple(c) not in present
        retried += att[s] > 1
    assert retried > 20                          # rho ~ 0.2: rejections exercised
    # f-sample zeros: kind 3
    fs, _, _, fa = orc.sample_export(t, 1, seed, rank, 0xFFFFFFFF, q, 0, 50, f_samples=True)
    for s in range(50):
        if fa[s] == 1:
            c = [t.lo[k] + _rmap(_words(orc, seed, s, rank, 3, 0, k // 2, 0xFFFFFFFF)[k % 2],
                                 t.hi[k] - t.lo[k]) for k in range(t.d)]
            assert tuple(fs[s]) == tuple(c)


def test_r11_gradient_and_estimate_use_the_exported_draws(orc):
    """The fused gradient consumes exactly the exported samples
    (nonzeros first, then zeros, slot order), and the loss estimate is the
    stratified sum over the kind-2/3 draws at iteration word 0xFFFFFFFF."""
    dims, t, _ = _rng_fixture(orc)
    A = orc.factor_init(4, dims, 3)
    seed, it, rank, p, q = 4242, 7, 1, 60, 70
    coords, y = orc.build_Y(t, A, "poisson", seed, rank, it, p, q)
    nz, _, _, _ = orc.sample_export(t, 0, seed, rank, it, p, 0, p)
    zz, _, _, _ = orc.sample_export(t, 1, seed, rank, it, q, 0, q)
    assert np.array_equal(coords, np.concatenate([nz, zz]))
    G, _, _ = orc.sampled_grad(t, A, "poisson", seed, rank, it, p, q)
    G2 = orc.mttkrp(t, A, coords, y)
    assert all(np.array_equal(a, b) for a, b in zip(G, G2))
    # loss estimate from the f-sample draws, summed here term by term
    fnz, fz = 90, 110
    est, _ = orc.loss_estimate(t, A, "poisson", seed, rank, fnz, fz)
    s1, _, _, _ = orc.sample_export(t, 0, seed, rank, 0xFFFFFFFF, fnz, 0, fnz, f_samples=True)
    s0, _, _, _ = orc.sample_export(t, 1, seed, rank, 0xFFFFFFFF, fz, 0, fz, f_samples=True)
    ss, sv = t.sorted()
    val = {tuple(c): x for c, x in zip(map(tuple, ss), sv)}
    tot = (t.nnz / fnz) * math.fsum(orc.loss_f("poisson", val[tuple(c)], orc.model_value(t, A, c)) for c in s1)
    tot += ((t.M - t.nnz) / fz) * math.fsum(orc.loss_f("poisson", 0.0, orc.model_value(t, A, c)) for c in s0)
    assert est == pytest.approx(tot, rel=1e-12)
