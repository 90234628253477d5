"""Pins for the oracle's RNG layer (reading R11): Philox KAT, range map, sampler draws."""
import numpy as np
import pytest
from conftest import GOLDEN

import gcp_synth


def test_philox_known_answers(orc):
    n = 0
    for line in (GOLDEN / "philox4x32_10_kat.txt").read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        v = [int(x, 16) for x in line.split()]
        assert orc.philox(v[0:4], v[4:6]) == v[6:10]
        n += 1
    assert n == 3


def test_range_map_endpoints_and_uniformity(orc):
    # floor(W n / 2^64): endpoints and the midpoint are fixed by the definition
    for n in (1, 7, 10_000, 4_821_207, 2 ** 40 + 3):
        assert orc.range_map(0, n) == 0
        assert orc.range_map(2 ** 64 - 1, n) == n - 1
        assert orc.range_map(2 ** 63, n) == n // 2
    # chi-square uniformity of mapped Philox words into 10 bins
    counts = np.zeros(10, int)
    for i in range(20000):
        o = orc.philox([i, 0, 0, 0], [12345, 0])
        W = o[0] | (o[1] << 32)
        counts[orc.range_map(W, 10)] += 1
    chi2 = ((counts - 2000) ** 2 / 2000).sum()
    assert chi2 < 27.9  # 9 dof, p = 0.001


def test_nonzero_draws_are_canonical_records(orc):
    subs, vals = gcp_synth.uniform_sparse((9, 8, 7), 120, seed=5)
    t = orc.Tensor((9, 8, 7), subs, vals)
    ss, sv = t.sorted()
    # canonical order is lexicographic with i_1 most significant (reading R15)
    assert [tuple(r) for r in ss] == sorted(tuple(r) for r in subs)
    e_subs, j, w, att = orc.sample_export(t, 0, seed=77, rank=0, it=3, n_stratum=500, first=0, count=500)
    assert (j >= 0).all() and (j < 120).all()
    assert (e_subs == ss[j]).all()
    assert np.allclose(w, 120 / 500) and (att == 1).all()
    # chi-square uniformity of j over 120 records from 24000 draws
    _, j2, _, _ = orc.sample_export(t, 0, seed=78, rank=0, it=0, n_stratum=24000, first=0, count=24000)
    cnt = np.bincount(j2, minlength=120)
    chi2 = ((cnt - 200) ** 2 / 200).sum()
    assert chi2 < 180  # 119 dof, p ~ 2e-4


def test_zero_draws_absent_and_acceptance_rate(orc):
    dims = (20, 30, 40)
    subs, vals = gcp_synth.uniform_sparse(dims, 2400, seed=1, values="counts")  # rho = 0.1
    t = orc.Tensor(dims, subs, vals)
    q = 20000
    zs, j, w, att = orc.sample_export(t, 1, seed=9, rank=0, it=0, n_stratum=q, first=0, count=q)
    assert (j == -1).all()
    assert all(not t.contains(c) for c in zs[:3000])
    S = set(map(tuple, subs))
    assert not any(tuple(c) in S for c in zs)
    assert np.allclose(w, (24000 - 2400) / q)
    # attempts ~ Geometric(1 - rho): acceptance fraction = q / sum(att) within 3 sigma
    acc = q / att.sum()
    sigma = np.sqrt(0.9 * 0.1 / att.sum())
    assert abs(acc - 0.9) < 3 * sigma + 1e-3
    # per-mode coordinate uniformity of the (accepted) zero draws
    for k, I in enumerate(dims):
        cnt = np.bincount(zs[:, k], minlength=I)
        exp = q / I
        chi2 = ((cnt - exp) ** 2 / exp).sum()
        assert chi2 < I + 5 * np.sqrt(2 * I)


def test_rejection_cap_and_no_zero_errors(orc):
    # full tensor: no zeros exist
    dims = (2, 2, 2)
    subs = np.array(np.unravel_index(np.arange(8), dims)).T
    t = orc.Tensor(dims, subs, np.ones(8))
    with pytest.raises(orc.OracleError) as e:
        orc.sample_export(t, 1, 1, 0, 0, 10, 0, 10)
    assert e.value.name == "E_NO_ZEROS"
    # one zero in 10^4 entries: P(1000 rejections) = (1-1e-4)^1000 ~ 0.9 -> cap hit
    dims = (10, 10, 100)
    lin = np.arange(10 * 10 * 100)[1:]
    subs = np.array(np.unravel_index(lin, dims)).T
    t = orc.Tensor(dims, subs, np.ones(len(lin)))
    with pytest.raises(orc.OracleError) as e:
        orc.sample_export(t, 1, 1, 0, 0, 10, 0, 10)
    assert e.value.name == "E_REJECT_CAP"


def test_ingest_errors(orc):
    with pytest.raises(orc.OracleError) as e:
        orc.Tensor((3, 3), np.array([[0, 1], [0, 1]]), np.array([1.0, 2.0]))
    assert e.value.name == "E_DUP"
    with pytest.raises(orc.OracleError) as e:
        orc.Tensor((3, 3), np.array([[0, 3]]), np.array([1.0]))
    assert e.value.name == "E_RANGE"
    with pytest.raises(orc.OracleError) as e:
        orc.Tensor((3, 3), np.array([[0, 1]]), np.array([np.nan]))
    assert e.value.name == "E_ARG"


def test_factor_init_uniform(orc):
    A = orc.factor_init(2002, (100, 50, 70), 8)
    allv = np.concatenate([a.ravel() for a in A])
    assert allv.min() >= 0 and allv.max() < 1
    assert abs(allv.mean() - 0.5) < 4 * np.sqrt(1 / 12 / allv.size)
    # element e of the concatenation uses Philox counter (lo32 e, hi32 e, 4<<28, 0)
    o = orc.philox([5, 0, 4 << 28, 0], [2002, 0])
    W0 = o[0] | (o[1] << 32)
    assert A[0].ravel()[5] == (W0 >> 11) * 2.0 ** -53
