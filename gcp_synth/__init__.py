"""Seeded synthetic inputs for GCP-Adam, shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no model value, loss,
gradient, sampling or Adam): it only manufactures data tensors with the
shape, density and skew of the paper's workloads and hands the
same arrays to both sides.

* ``chi_kolda``  -- Chi-Kolda-style count tensor, "adapted from Chi and Kolda
  ... scales random factor matrix entries to be much larger":
  random factors with 10% of the entries of every column boosted 10x, columns
  normalised to sum 1, lambda_r = 1/R; each draw picks r ~ lambda, then
  i_k ~ A^(k)(:, r); duplicate coordinates merge and their count is the value.
* ``uniform_sparse`` -- distinct uniformly random coordinates, for tiny tests.
* ``CONFIGS`` -- the five BASELINE.json configs (reading R22 for the shapes).

torch is used only as a fast seeded RNG/sort engine (CPU or CUDA); a given
(seed, device) always yields the same tensor.
"""
from __future__ import annotations

import math

import numpy as np
import torch

# BASELINE.json configs.  nnz is the target count.
CONFIGS = {
    "c1": dict(dims=(20, 30, 40), nnz=2400, R=4, loss="poisson", s=1000, f=2000),
    "c2": dict(dims=(10000, 10000, 10000), nnz=100_000_000, R=16, loss="poisson",
               s=10_000_000, f=10_000_000),
    "c3": dict(dims=(1605, 4198, 1631, 4209, 868131), nnz=1_698_825, R=10, loss="bernoulli",
               s=1_000_000, f=1_000_000),
    "c4": dict(dims=(4_821_207, 1_774_269, 1_805_187), nnz=1_741_809_018, R=16, loss="gaussian",
               s=10_000_000, f=10_000_000),
    "c5": dict(dims=(8_211_298, 176_962, 8_116_559), nnz=4_687_474_081, R=32, loss="poisson",
               s=100_000_000, f=10_000_000),
}
SEEDS = {c: dict(data=1000 + i, model=2000 + i, sample=3000 + i)
         for i, c in enumerate(["c1", "c2", "c3", "c4", "c5"], start=1)}


def _gen(seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _lin_keys(subs, dims):
    """Mixed-radix linear index (int64) used only to merge duplicate draws."""
    key = subs[:, 0].clone()
    for k in range(1, len(dims)):
        key = key * int(dims[k]) + subs[:, k]
    return key


def _unlin(keys, dims):
    d = len(dims)
    out = torch.empty((keys.numel(), d), dtype=torch.int64, device=keys.device)
    rem = keys.clone()
    for k in range(d - 1, -1, -1):
        out[:, k] = rem % int(dims[k])
        rem = rem // int(dims[k])
    return out


def _merge2(hi, lo, cnt):
    """Merge duplicate (hi, lo) keys, summing counts; result sorted by (hi, lo).
    Keeps the dtypes of hi and cnt (int32 in the compact billion-scale parts)."""
    o = torch.argsort(lo, stable=True)
    hi, lo, cnt = hi[o], lo[o], cnt[o]
    o = torch.argsort(hi, stable=True)
    hi, lo, cnt = hi[o], lo[o], cnt[o]
    del o
    new = torch.ones(hi.numel(), dtype=torch.bool, device=hi.device)
    new[1:] = (hi[1:] != hi[:-1]) | (lo[1:] != lo[:-1])
    seg = torch.cumsum(new, 0) - 1
    cu = torch.zeros(int(seg[-1]) + 1 if seg.numel() else 0, dtype=torch.int64, device=hi.device)
    cu.index_add_(0, seg, cnt.long())
    return hi[new], lo[new], cu.to(cnt.dtype)


def chi_kolda(dims, nnz, R, seed, loss="poisson", device="cpu", boost_frac=0.1, boost=10.0,
              tol=0.005, max_rounds=64, force_wide=False, block=None, allreduce=None, out_device=None):
    """Return (subs int64 [N, d], vals float64 [N]) as torch tensors on `device`.

    Duplicate draws merge on an int64 mixed-radix key when prod(dims) < 2^62,
    else on the pair (i_1, key of the other modes) (needs prod(dims[1:]) < 2^63).

    block = (lo, hi): keep only the entries with lo_k <= i_k < hi_k (one rank's
    block of a medium-grained grid) without materialising the rest.  Every rank
    consumes the identical draw stream, so the blocks of all ranks partition the
    one global tensor; `allreduce(int) -> int` sums the kept distinct counts over
    the ranks, so the top-up test sees the global count.  Only the rare thinning
    step (an overshoot beyond nnz * (1 + tol)) and the shuffle order then depend
    on the block.

    out_device: where the returned tensors live (default `device`).  On the
    billion-scale path with out_device="cpu" each finished i_1 partition moves to
    host memory as it is built, so a tensor larger than the device's memory (c5
    at one GPU: 4.69e9 nonzeros, 150 GB of int64 + fp64 COO) can be generated
    on the device.  The partitions are kept compact while merging (i_1 and the
    counts as int32), which changes no value."""
    out_device = device if out_device is None else out_device
    dims = [int(i) for i in dims]
    wide = force_wide or block is not None or math.prod(dims) >= 2 ** 62
    assert not wide or math.prod(dims[1:]) < 2 ** 63
    assert nnz <= math.prod(dims)
    g = _gen(seed, device)
    cdfs = []
    for I in dims:
        A = torch.rand((R, I), generator=g, device=device, dtype=torch.float64)
        nb = max(1, int(round(boost_frac * I)))
        for r in range(R):
            idx = torch.randperm(I, generator=g, device=device)[:nb]
            A[r, idx] *= boost
        A /= A.sum(dim=1, keepdim=True)
        c = torch.cumsum(A, dim=1)
        c[:, -1] = 1.0
        cdfs.append((c + torch.arange(R, device=device, dtype=torch.float64)[:, None]).reshape(-1))
        del A, c
    lo_target = int(math.floor(nnz * (1 - tol)))
    if not wide:
        keys = torch.empty(0, dtype=torch.int64, device=device)
        counts = torch.empty(0, dtype=torch.int64, device=device)
        want = nnz
        for _ in range(max_rounds):
            n_draw = max(1024, int((want - keys.numel()) * 1.02) + 64)
            cols = _draw(cdfs, dims, R, n_draw, g, device)
            nk = _lin_keys(torch.stack(cols, 1), dims)
            del cols
            allk = torch.cat([keys, nk])
            allc = torch.cat([counts, torch.ones_like(nk)])
            del nk
            keys, inv = torch.unique(allk, sorted=True, return_inverse=True)
            counts = torch.zeros_like(keys).index_add_(0, inv, allc)
            del allk, allc, inv
            if keys.numel() >= lo_target:
                break
        if keys.numel() > nnz * (1 + tol):
            # deterministic thinning to the tolerance band (keeps sorted order)
            perm = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
            perm, _ = torch.sort(perm)
            keys, counts = keys[perm], counts[perm]
        # shuffle so that ingest sees an unsorted list, like a file would be
        perm = torch.randperm(keys.numel(), generator=g, device=device)
        keys, counts = keys[perm], counts[perm]
        del perm
        subs = _unlin(keys, dims)
        del keys
    else:
        # Billion-scale path: draws arrive in rounds of <= 4e8 and are split into
        # i_1-range partitions (duplicates share i_1) of < 2^31 entries each, so
        # every sort stays below 2^31 elements.
        blo, bhi = (list(block[0]), list(block[1])) if block is not None else ([0] * len(dims), dims)
        nparts = max(1, -(-nnz // 200_000_000))
        edges = [int(blo[0]) + (int(bhi[0]) - int(blo[0])) * j // nparts for j in range(nparts + 1)]
        # compact partitions: i_1 (< 2^31) and the counts as int32, the key of the
        # other modes as int64 (16 B per distinct entry while merging)
        assert dims[0] < 2 ** 31
        parts = [(torch.empty(0, dtype=torch.int32, device=device), torch.empty(0, dtype=torch.int64, device=device),
                  torch.empty(0, dtype=torch.int32, device=device)) for _ in range(nparts)]
        total = 0
        for _ in range(max_rounds):
            left = max(1024, int((nnz - total) * 1.02) + 64)
            while left > 0:
                n_draw = min(left, 400_000_000)
                left -= n_draw
                cols = _draw(cdfs, dims, R, n_draw, g, device)
                if block is not None:
                    m = torch.ones(n_draw, dtype=torch.bool, device=device)
                    for k in range(len(dims)):
                        m &= (cols[k] >= int(blo[k])) & (cols[k] < int(bhi[k]))
                    cols = [c[m] for c in cols]
                    del m
                nlo = cols[1].clone()
                for k in range(2, len(dims)):
                    nlo = nlo * dims[k] + cols[k]
                nhi = cols[0]
                del cols
                pid = torch.bucketize(nhi, torch.tensor(edges[1:-1], device=device), right=True)
                for j in range(nparts):
                    m = pid == j
                    ph, pl, pc = parts[j]
                    parts[j] = _merge2(torch.cat([ph, nhi[m].int()]), torch.cat([pl, nlo[m]]),
                                       torch.cat([pc, torch.ones(int(m.sum()), dtype=torch.int32, device=device)]))
                del nhi, nlo, pid
            total = sum(p[0].numel() for p in parts)
            if allreduce is not None:
                total = int(allreduce(total))
            if total >= lo_target:
                break
        keep = nnz / total if total > nnz * (1 + tol) else None
        subs_l, cnt_l = [], []
        to_host = torch.device(out_device) != torch.device(device)
        if to_host:   # filled partition by partition; capacity bound: the tolerance band
            cap = int(nnz * (1 + tol)) + 1_000_000
            subs = torch.empty((cap, len(dims)), dtype=torch.int64, device=out_device)
            counts = torch.empty(cap, dtype=torch.float64, device=out_device)   # the values, filled directly
            o = 0
        for j in range(nparts):
            ph, pl, pc = parts[j]
            parts[j] = None
            if keep is not None:   # Bernoulli thinning to the tolerance band
                m = torch.rand(ph.numel(), generator=g, device=device) < keep
                ph, pl, pc = ph[m], pl[m], pc[m]
            perm = torch.randperm(ph.numel(), generator=g, device=device)   # shuffle within the partition
            ph, pl, pc = ph[perm], pl[perm], pc[perm]
            sj = torch.empty((ph.numel(), len(dims)), dtype=torch.int64, device=device)
            sj[:, 0] = ph
            sj[:, 1:] = _unlin(pl, dims[1:])
            if to_host:
                n = sj.shape[0]
                assert o + n <= cap
                subs[o:o + n] = sj
                counts[o:o + n] = pc.double() if loss != "bernoulli" else 1.0
                o += n
            else:
                subs_l.append(sj)
                cnt_l.append(pc.long())
            del ph, pl, perm, sj
        if to_host:
            subs, counts = subs[:o], counts[:o]
        else:
            subs = torch.cat(subs_l)
            counts = torch.cat(cnt_l)
        del subs_l, cnt_l
    if counts.dtype == torch.float64:   # host-assembled billion-scale values (already final)
        vals = counts
    elif loss == "bernoulli":
        vals = torch.ones(counts.numel(), dtype=torch.float64, device=counts.device)
    else:
        vals = counts.double()
    if not wide and torch.device(out_device) != torch.device(device):
        subs, vals = subs.to(out_device), vals.to(out_device)
    return subs, vals


def _draw(cdfs, dims, R, n, g, device):
    """n Chi-Kolda draws: r ~ uniform(R) (lambda_r = 1/R), then i_k ~ A^(k)(:, r)
    by inverse CDF."""
    r = torch.randint(0, R, (n,), generator=g, device=device)
    cols = []
    for k, I in enumerate(dims):
        u = torch.rand(n, generator=g, device=device, dtype=torch.float64)
        u += r
        i = torch.searchsorted(cdfs[k], u, right=True)
        del u
        i -= r * I
        cols.append(i.clamp_(0, I - 1))
    return cols


def uniform_sparse(dims, nnz, seed, values="normal"):
    """Distinct uniform random coordinates (numpy) for tiny oracle tests."""
    rng = np.random.default_rng(seed)
    M = math.prod(dims)
    lin = rng.choice(M, size=nnz, replace=False)
    subs = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
    if values == "normal":
        vals = rng.normal(size=nnz)
    elif values == "counts":
        vals = rng.integers(1, 5, size=nnz).astype(np.float64)
    elif values == "ones":
        vals = np.ones(nnz)
    else:
        raise ValueError(values)
    return subs, vals


def random_factors(dims, R, seed, low=0.0, high=1.0):
    rng = np.random.default_rng(seed)
    return [rng.uniform(low, high, size=(int(I), R)) for I in dims]


def config_tensor(name, device="cpu"):
    """The data tensor of config `name` with its data seed (torch tensors)."""
    c = CONFIGS[name]
    return chi_kolda(c["dims"], c["nnz"], c["R"], SEEDS[name]["data"], c["loss"], device=device)
