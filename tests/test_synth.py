"""The seeded generator (gcp_synth, no method arithmetic): determinism, the
target nnz band, distinct coordinates, and the wide-key merge path agreeing
with the int64-key path."""
import math

import numpy as np
import torch

import gcp_synth


def test_chi_kolda_deterministic_distinct_in_band():
    dims = (60, 50, 40)
    s1, v1 = gcp_synth.chi_kolda(dims, 5000, 3, 11)
    s2, v2 = gcp_synth.chi_kolda(dims, 5000, 3, 11)
    assert torch.equal(s1, s2) and torch.equal(v1, v2)
    assert abs(len(v1) - 5000) <= 0.005 * 5000
    lin = (s1[:, 0] * 50 + s1[:, 1]) * 40 + s1[:, 2]
    assert torch.unique(lin).numel() == len(lin)
    assert (v1 >= 1).all() and v1.sum() >= len(v1)
    for k, I in enumerate(dims):
        assert s1[:, k].min() >= 0 and s1[:, k].max() < I


def test_wide_key_path_matches_narrow():
    """Same draws, same merge: with a tolerance band wide enough that neither
    path thins, both yield the same set of (coordinates, count)."""
    dims = (300, 200, 100)
    a = gcp_synth.chi_kolda(dims, 20000, 4, 3, tol=0.05)
    b = gcp_synth.chi_kolda(dims, 20000, 4, 3, tol=0.05, force_wide=True)

    def canon(sv):
        s, v = sv
        key = (s[:, 0] * 200 + s[:, 1]) * 100 + s[:, 2]
        o = torch.argsort(key)
        return key[o], v[o]
    ka, va = canon(a)
    kb, vb = canon(b)
    assert torch.equal(ka, kb) and torch.equal(va, vb)


def test_wide_shape_lbnl_like():
    dims = gcp_synth.CONFIGS["c3"]["dims"]
    assert math.prod(dims) > 2 ** 64
    s, v = gcp_synth.chi_kolda(dims, 5000, 10, 7, loss="bernoulli")
    assert (v == 1).all() and abs(len(v) - 5000) <= 25
    rows = {tuple(r) for r in s.tolist()}
    assert len(rows) == len(v)


def test_block_generation_partitions_the_global_tensor():
    """Per-rank block generation (bench at N > 1): four concurrent 'ranks' of a
    2x1x2 grid, summing their kept counts through a barrier-based allreduce,
    reproduce exactly the blocks of the whole tensor (tolerance band wide
    enough that nothing is thinned)."""
    import threading
    dims = (300, 200, 100)
    full = gcp_synth.chi_kolda(dims, 20000, 4, 3, tol=0.05, force_wide=True)
    blocks = [([0, 0, 0], [150, 200, 50]), ([0, 0, 50], [150, 200, 100]),
              ([150, 0, 0], [300, 200, 50]), ([150, 0, 50], [300, 200, 100])]
    bar = threading.Barrier(4)
    slots, out = [0] * 4, [None] * 4

    def rank(w):
        def allreduce(x):
            slots[w] = x
            bar.wait()
            t = sum(slots)
            bar.wait()
            return t
        out[w] = gcp_synth.chi_kolda(dims, 20000, 4, 3, tol=0.05, block=blocks[w], allreduce=allreduce)

    th = [threading.Thread(target=rank, args=(w,)) for w in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()

    def canon(s, v):
        key = (s[:, 0] * 200 + s[:, 1]) * 100 + s[:, 2]
        o = torch.argsort(key)
        return key[o], v[o]
    fs, fv = full
    for w, (lo, hi) in enumerate(blocks):
        m = torch.ones(len(fv), dtype=torch.bool)
        for k in range(3):
            m &= (fs[:, k] >= lo[k]) & (fs[:, k] < hi[k])
        kf, vf = canon(fs[m], fv[m])
        kb, vb = canon(*out[w])
        assert torch.equal(kf, kb) and torch.equal(vf, vb), w
    assert sum(len(o[1]) for o in out) == len(fv)
