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


def chi_kolda(dims, nnz, R, seed, loss="poisson", device="cpu", boost_frac=0.1, boost=10.0,
              tol=0.005, max_rounds=64):
    """Return (subs int64 [N, d], vals float64 [N]) as torch tensors on `device`.

    Requires prod(dims) < 2^63 (the merge key is int64)."""
    dims = [int(i) for i in dims]
    assert math.prod(dims) < 2 ** 63, "merge key would overflow int64"
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
    keys = torch.empty(0, dtype=torch.int64, device=device)
    counts = torch.empty(0, dtype=torch.int64, device=device)
    lo_target = int(math.floor(nnz * (1 - tol)))
    want = nnz
    for _ in range(max_rounds):
        n_draw = max(1024, int((want - keys.numel()) * 1.02) + 64)
        r = torch.randint(0, R, (n_draw,), generator=g, device=device)
        cols = []
        for k, I in enumerate(dims):
            u = torch.rand(n_draw, generator=g, device=device, dtype=torch.float64) + r.double()
            i = torch.searchsorted(cdfs[k], u, right=True) - r * I
            cols.append(i.clamp_(0, I - 1))
        del r
        nk = _lin_keys(torch.stack(cols, 1), dims)
        del cols
        allk = torch.cat([keys, nk])
        allc = torch.cat([counts, torch.ones_like(nk)])
        keys, inv = torch.unique(allk, sorted=True, return_inverse=True)
        counts = torch.zeros_like(keys).index_add_(0, inv, allc)
        del allk, allc, inv, nk
        if keys.numel() >= lo_target:
            break
        # far below target (dense, collision-heavy tensor): draw more next round
        want = nnz
    if keys.numel() > nnz * (1 + tol):
        # deterministic thinning to the tolerance band (keeps sorted order)
        perm = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
        perm, _ = torch.sort(perm)
        keys, counts = keys[perm], counts[perm]
    # shuffle so that ingest sees an unsorted list, like a file would be
    perm = torch.randperm(keys.numel(), generator=g, device=device)
    keys, counts = keys[perm], counts[perm]
    subs = _unlin(keys, dims)
    if loss == "bernoulli":
        vals = torch.ones(keys.numel(), dtype=torch.float64, device=device)
    else:
        vals = counts.double()
    return subs, vals


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
