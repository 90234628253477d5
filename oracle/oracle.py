"""ctypes marshalling for gcp_oracle.c plus the paper's multi-rank loops.

TEST INFRASTRUCTURE ONLY (see package docstring).  All per-sample arithmetic
is in gcp_oracle.c; the Python here strings C calls together in the order of
the paper's algorithms:

* ``sync_gradient``   -- Alg. 2: per-rank sampled gradients summed
  over ranks in rank-major order (readings R13, R21).
* ``fit``             -- the epoch loop with annealing (P:868-869, P:1410-1412,
  reading R20) around Alg. 2 (sync), Alg. 3 (LocalSGD, reading R16)
  or Alg. 4 (FedAdam, reading R17).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "gcp_oracle.c"
_LIB = _HERE / "liboracle.so"

LOSSES = {"gaussian": 0, "poisson": 1, "bernoulli": 2}
STRATEGIES = {"stratified": 0, "semi": 1}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_RANGE", 3: "E_DUP", 4: "E_NO_NONZEROS",
          5: "E_NO_ZEROS", 6: "E_REJECT_CAP", 9: "E_OOM"}


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"oracle {self.name} {msg}")


def build(force: bool = False) -> Path:
    """Compile gcp_oracle.c (plain -O2, no fast-math)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
                               "-fno-fast-math", "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(_LIB))
        i64p, dp, u32p, i32p = (C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_int32))
        vp = C.c_void_p
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_range_map.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_range_map.restype = C.c_uint64
        L.orc_tensor_new.argtypes = [C.c_int, i64p, i64p, i64p, C.c_int64, i64p, dp, C.POINTER(vp)]
        L.orc_tensor_free.argtypes = [vp]
        L.orc_tensor_nnz.argtypes = [vp]
        L.orc_tensor_nnz.restype = C.c_int64
        L.orc_tensor_M.argtypes = [vp]
        L.orc_tensor_M.restype = C.c_double
        L.orc_tensor_sorted.argtypes = [vp, i64p, dp]
        L.orc_tensor_contains.argtypes = [vp, i64p]
        L.orc_model_value.argtypes = [vp, C.c_int, dp, dp, i64p]
        L.orc_model_value.restype = C.c_double
        for f in ("orc_loss_f", "orc_loss_df"):
            getattr(L, f).argtypes = [C.c_int, C.c_double, C.c_double]
            getattr(L, f).restype = C.c_double
        L.orc_loss_lower.argtypes = [C.c_int]
        L.orc_loss_lower.restype = C.c_double
        L.orc_alloc_count.argtypes = [C.c_int64, C.c_int, C.c_int]
        L.orc_alloc_count.restype = C.c_int64
        L.orc_sample_export.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                        i64p, i64p, dp, i32p, i64p]
        L.orc_mttkrp.argtypes = [vp, C.c_int, dp, dp, C.c_int64, i64p, dp, dp]
        L.orc_build_Y.argtypes = [vp, C.c_int, dp, dp, C.c_int, C.c_int, C.c_uint64, C.c_uint32,
                                  C.c_uint32, C.c_int64, C.c_int64, i64p, dp, i64p]
        L.orc_sampled_grad.argtypes = [vp, C.c_int, dp, dp, C.c_int, C.c_int, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_int64, C.c_int64, dp, dp, dp, dp, i64p]
        L.orc_loss_estimate.argtypes = [vp, C.c_int, dp, dp, C.c_int, C.c_uint64, C.c_uint32,
                                        C.c_int64, C.c_int64, dp, dp, i64p]
        L.orc_sampled_grad_par.argtypes = [vp, C.c_int, dp, dp, C.c_int, C.c_int, C.c_uint64, C.c_uint32,
                                           C.c_uint32, C.c_int64, C.c_int64, dp, dp, C.c_int]
        L.orc_loss_estimate_par.argtypes = [vp, C.c_int, dp, dp, C.c_int, C.c_uint64, C.c_uint32,
                                            C.c_int64, C.c_int64, dp, C.c_int]
        L.orc_adam_par.argtypes = [C.c_int64, dp, dp, dp, dp, C.c_int64, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_int]
        L.orc_full_loss.argtypes = [vp, C.c_int, dp, dp, C.c_int, dp]
        L.orc_full_grad.argtypes = [vp, C.c_int, dp, dp, C.c_int, dp]
        L.orc_adam.argtypes = [C.c_int64, dp, dp, dp, dp, C.c_int64, C.c_double, C.c_double,
                               C.c_double, C.c_double, C.c_double]
        L.orc_factor_init.argtypes = [C.c_uint64, C.c_int, i64p, C.c_int, dp]
        L.orc_grid_plan.argtypes = [C.c_int, C.c_int, i64p, C.POINTER(C.c_int)]
        L.orc_grid_plan.restype = C.c_double
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(st, msg=""):
    if st != 0:
        raise OracleError(st, msg)


# ---------------------------------------------------------------- primitives
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(o, C.c_uint32))
    return [int(v) for v in o]


def range_map(W, n):
    return int(lib().orc_range_map(W, n))


def loss_f(loss, x, m):
    return lib().orc_loss_f(LOSSES[loss], float(x), float(m))


def loss_df(loss, x, m):
    return lib().orc_loss_df(LOSSES[loss], float(x), float(m))


def loss_lower(loss):
    return lib().orc_loss_lower(LOSSES[loss])


def alloc_count(total, P, w):
    return int(lib().orc_alloc_count(total, P, w))


def factor_init(seed, dims, R):
    """Global factors A^(k) (I_k x R, fp64) per reading R12."""
    dims_a = _i64(dims)
    out = np.zeros(int(sum(int(i) for i in dims) * R), dtype=np.float64)
    lib().orc_factor_init(seed, len(dims), _p(dims_a, C.c_int64), R, _p(out, C.c_double))
    res, off = [], 0
    for I in dims:
        res.append(out[off:off + int(I) * R].reshape(int(I), R).copy())
        off += int(I) * R
    return res


def grid_plan(P, dims):
    dims_a = _i64(dims)
    g = (C.c_int * len(dims))()
    obj = lib().orc_grid_plan(P, len(dims), _p(dims_a, C.c_int64), g)
    return tuple(int(v) for v in g), obj


def rank_coords(rank, grid):
    """rank <-> (b_1..b_d), row-major with b_1 slowest (reading R14)."""
    b = []
    for n in reversed(grid):
        b.append(rank % n)
        rank //= n
    return tuple(reversed(b))


def block_bounds(dims, grid, rank):
    """c_k = ceil(I_k/N_k); lo = b c_k; hi = min((b+1) c_k, I_k) (reading R14)."""
    b = rank_coords(rank, grid)
    lo, hi = [], []
    for I, n, bk in zip(dims, grid, b):
        c = -(-int(I) // n)
        lo.append(min(bk * c, int(I)))
        hi.append(min((bk + 1) * c, int(I)))
    return lo, hi


# ---------------------------------------------------------------- tensor
class Tensor:
    """One rank's block of the COO tensor, sorted lexicographically."""

    def __init__(self, dims, subs, vals, lo=None, hi=None):
        self.dims = [int(i) for i in dims]
        self.d = len(self.dims)
        self.lo = [0] * self.d if lo is None else [int(v) for v in lo]
        self.hi = list(self.dims) if hi is None else [int(v) for v in hi]
        subs = _i64(subs).reshape(-1, self.d) if len(subs) else np.zeros((0, self.d), np.int64)
        vals = _f64(vals)
        h = C.c_void_p()
        dims_a, lo_a, hi_a = _i64(self.dims), _i64(self.lo), _i64(self.hi)
        _check(lib().orc_tensor_new(self.d, _p(dims_a, C.c_int64), _p(lo_a, C.c_int64),
                                    _p(hi_a, C.c_int64), len(vals), _p(subs, C.c_int64),
                                    _p(vals, C.c_double), C.byref(h)), "tensor_new")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_tensor_free(self._h)
            self._h = None

    @property
    def nnz(self):
        return int(lib().orc_tensor_nnz(self._h))

    @property
    def M(self):
        """prod_k (hi_k - lo_k) as an exact Python int."""
        return math.prod(h - l for l, h in zip(self.lo, self.hi))

    def sorted(self):
        n = self.nnz
        s = np.zeros((n, self.d), np.int64)
        v = np.zeros(n, np.float64)
        lib().orc_tensor_sorted(self._h, _p(s, C.c_int64), _p(v, C.c_double))
        return s, v

    def contains(self, coords):
        c = _i64(coords)
        return bool(lib().orc_tensor_contains(self._h, _p(c, C.c_int64)))

    def block_rows(self, A):
        """Flat fp64 block rows of global factors A (list of I_k x R)."""
        return np.concatenate([np.asarray(A[k], np.float64)[self.lo[k]:self.hi[k]].ravel()
                               for k in range(self.d)])

    def split_rows(self, flat, R):
        out, off = [], 0
        for k in range(self.d):
            n = (self.hi[k] - self.lo[k]) * R
            out.append(flat[off:off + n].reshape(-1, R))
            off += n
        return out


def _lam(lam, R):
    return _f64(np.ones(R) if lam is None else lam)


def model_value(t, A, coords, lam=None):
    R = A[0].shape[1]
    Af, la, c = _f64(t.block_rows(A)), _lam(lam, R), _i64(coords)
    return lib().orc_model_value(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), _p(c, C.c_int64))


def sample_export(t, stratum, seed, rank, it, n_stratum, first, count,
                  strategy="stratified", f_samples=False):
    """Entries of Y~ for slots [first, first+count) of one stratum (0 nz, 1 zero)."""
    subs = np.zeros((count, t.d), np.int64)
    j = np.zeros(count, np.int64)
    w = np.zeros(count, np.float64)
    att = np.zeros(count, np.int32)
    err = C.c_int64(-1)
    st = lib().orc_sample_export(t._h, STRATEGIES[strategy], stratum, seed, rank, it,
                                 int(f_samples), n_stratum, first, count, _p(subs, C.c_int64),
                                 _p(j, C.c_int64), _p(w, C.c_double), _p(att, C.c_int32),
                                 C.byref(err))
    _check(st, f"slot {err.value}")
    return subs, j, w, att


def sampled_grad(t, A, loss, seed, rank, it, p_w, q_w, strategy="stratified", lam=None,
                 with_scale=True, loss_scale=False):
    """Fused Sampling-MTTKRP for one rank.  Returns (G, S, sampled loss)
    with G, S lists of block-row matrices; with loss_scale=True also the
    rounding scale sum |w f| of the sampled loss (tolerance only, C18)."""
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    G = np.zeros_like(Af)
    S = np.zeros_like(Af) if with_scale else None
    ls, lsc = C.c_double(0), C.c_double(0)
    err = C.c_int64(-1)
    st = lib().orc_sampled_grad(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                                STRATEGIES[strategy], seed, rank, it, p_w, q_w,
                                _p(G, C.c_double), _p(S, C.c_double) if with_scale else None,
                                C.byref(ls), C.byref(lsc) if loss_scale else None, C.byref(err))
    _check(st, f"slot {err.value}")
    out = (t.split_rows(G, R), (t.split_rows(S, R) if with_scale else None), ls.value)
    return out + (lsc.value,) if loss_scale else out


def build_Y(t, A, loss, seed, rank, it, p_w, q_w, strategy="stratified", lam=None):
    """Non-fused step 1: explicit Y~ as (coords, values)."""
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    coords = np.zeros((p_w + q_w, t.d), np.int64)
    y = np.zeros(p_w + q_w, np.float64)
    err = C.c_int64(-1)
    st = lib().orc_build_Y(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                           STRATEGIES[strategy], seed, rank, it, p_w, q_w,
                           _p(coords, C.c_int64), _p(y, C.c_double), C.byref(err))
    _check(st, f"slot {err.value}")
    return coords, y


def mttkrp(t, A, coords, y, lam=None):
    """Sparse MTTKRP of an entry list over block rows (Eq. gcp-gradient)."""
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    c, yy = _i64(coords).reshape(-1, t.d), _f64(y)
    G = np.zeros_like(Af)
    lib().orc_mttkrp(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), len(yy),
                     _p(c, C.c_int64), _p(yy, C.c_double), _p(G, C.c_double))
    return t.split_rows(G, R)


def loss_estimate(t, A, loss, seed, rank, f_nz, f_z, lam=None):
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    est, sc, err = C.c_double(0), C.c_double(0), C.c_int64(-1)
    st = lib().orc_loss_estimate(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                                 seed, rank, f_nz, f_z, C.byref(est), C.byref(sc), C.byref(err))
    _check(st, f"slot {err.value}")
    return est.value, sc.value


def full_loss(t, A, loss, lam=None):
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    out = C.c_double(0)
    _check(lib().orc_full_loss(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                               C.byref(out)), "full_loss guard")
    return out.value


def full_grad(t, A, loss, lam=None):
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    G = np.zeros_like(Af)
    _check(lib().orc_full_grad(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                               _p(G, C.c_double)), "full_grad guard")
    return t.split_rows(G, R)


# ---------------------------------------------------------------- OpenMP timing variants
def host_threads():
    """Host threads this process may use (the CPU-baseline core count)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def sampled_grad_par(t, A, loss, seed, rank, it, p_w, q_w, strategy="stratified", lam=None, nthreads=None):
    """OpenMP variant of sampled_grad (timing only): same
    draws, thread-private G reduced in thread order.  Returns (G, sampled loss)."""
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    G = np.zeros_like(Af)
    ls = C.c_double(0)
    st = lib().orc_sampled_grad_par(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                                    STRATEGIES[strategy], seed, rank, it, p_w, q_w, _p(G, C.c_double),
                                    C.byref(ls), nthreads or host_threads())
    _check(st)
    return t.split_rows(G, R), ls.value


def loss_estimate_par(t, A, loss, seed, rank, f_nz, f_z, lam=None, nthreads=None):
    R = A[0].shape[1]
    Af, la = _f64(t.block_rows(A)), _lam(lam, R)
    est = C.c_double(0)
    st = lib().orc_loss_estimate_par(t._h, R, _p(la, C.c_double), _p(Af, C.c_double), LOSSES[loss],
                                     seed, rank, f_nz, f_z, C.byref(est), nthreads or host_threads())
    _check(st)
    return est.value


def adam_par(A, G, B, Cm, t, alpha, beta1=0.9, beta2=0.999, eps=1e-8, lower=-math.inf, nthreads=None):
    lib().orc_adam_par(A.size, _p(A, C.c_double), _p(G, C.c_double), _p(B, C.c_double),
                       _p(Cm, C.c_double), t, alpha, beta1, beta2, eps, lower, nthreads or host_threads())


def poisson_exact_grad(subs, vals, A, lam=None, chunk=4_000_000):
    """Exact gradient dF/dA^(k) of the Poisson GCP objective (P:282-296 with the
    loss of reading R3) at any scale, in O(N d R): f'(0, m) = 1 for every entry,
    so summing over all M entries gives
        G^(k)[i, r] = lam_r prod_{j != k} colsum_r(A^(j))
                      - sum_{nonzeros with i_k = i} x / (m + eps) lam_r prod_{j != k} A^(j)[i_j, r]
    (SURVEY C17 "Poisson identity"; pinned against enumeration in
    tests/test_oracle_math.py).  Global coordinates and global factors; fp64."""
    d, R = len(A), A[0].shape[1]
    lam = np.ones(R) if lam is None else np.asarray(lam, np.float64)
    A = [np.asarray(a, np.float64) for a in A]
    cs = [a.sum(axis=0) for a in A]
    G = []
    for k in range(d):
        dense = lam.copy()
        for j in range(d):
            if j != k:
                dense = dense * cs[j]
        G.append(np.tile(dense, (A[k].shape[0], 1)))
    subs = np.asarray(subs)
    vals = np.asarray(vals, np.float64)
    for c0 in range(0, len(vals), chunk):
        sb = subs[c0:c0 + chunk].astype(np.int64)
        rows = [A[k][sb[:, k]] for k in range(d)]
        full = lam * np.prod(rows, axis=0)                       # lam_r prod_k a_k[r]
        m = full.sum(axis=1)
        y = -vals[c0:c0 + chunk] / (m + 1e-10)
        for k in range(d):
            others = lam * np.prod([rows[j] for j in range(d) if j != k], axis=0)   # no division
            z = y[:, None] * others
            for r in range(R):
                G[k][:, r] += np.bincount(sb[:, k], weights=z[:, r], minlength=A[k].shape[0])
    return G


def adam(A, G, B, Cm, t, alpha, beta1=0.9, beta2=0.999, eps=1e-8, lower=-math.inf):
    """Alg. 1 in place on flat fp64 arrays; t = step number after increment."""
    for a in (A, G, B, Cm):
        assert a.dtype == np.float64 and a.flags.c_contiguous and a.size == A.size
    lib().orc_adam(A.size, _p(A, C.c_double), _p(G, C.c_double), _p(B, C.c_double),
                   _p(Cm, C.c_double), t, alpha, beta1, beta2, eps, lower)


# ---------------------------------------------------------------- multi-rank
def split_blocks(dims, subs, vals, P, grid=None):
    """Medium-grained partition: per-rank Tensor blocks."""
    if grid is None:
        grid, _ = grid_plan(P, dims)
    subs = _i64(subs).reshape(-1, len(dims))
    vals = _f64(vals)
    blocks = []
    for w in range(P):
        lo, hi = block_bounds(dims, grid, w)
        m = np.ones(len(vals), bool)
        for k in range(len(dims)):
            m &= (subs[:, k] >= lo[k]) & (subs[:, k] < hi[k])
        blocks.append(Tensor(dims, subs[m], vals[m], lo, hi))
    return blocks, grid


def local_counts(t, total_nz, total_z, P, w, stratified=True):
    """Per-rank sample counts (reading R13) with the empty-strata rule of
    SURVEY §8(c) C4: a block without nonzeros (zeros) draws none of them."""
    p = alloc_count(total_nz, P, w) if t.nnz > 0 else 0
    q = alloc_count(total_z, P, w) if t.M > t.nnz else 0
    return p, q


def sync_gradient(blocks, A, loss, seed, it, p, q, strategy="stratified", lam=None):
    """Alg. 2 lines 2-3: each rank's sampled gradient, summed into the global
    G^(k) in rank-major order.  Returns (G, S, sampled loss)."""
    P = len(blocks)
    G = [np.zeros_like(a, dtype=np.float64) for a in A]
    S = [np.zeros_like(a, dtype=np.float64) for a in A]
    ls = 0.0
    for w, t in enumerate(blocks):
        pw, qw = local_counts(t, p, q, P, w)
        Gw, Sw, lw = sampled_grad(t, A, loss, seed, w, it, pw, qw, strategy, lam)
        for k in range(t.d):
            G[k][t.lo[k]:t.hi[k]] += Gw[k]
            S[k][t.lo[k]:t.hi[k]] += Sw[k]
        ls += lw
    return G, S, ls


def sync_loss_estimate(blocks, A_of_rank, loss, seed, f_nz, f_z, lam=None):
    """Sum over ranks of each block's stratified estimate (reading R19).
    A_of_rank(w) gives the factors rank w evaluates with."""
    P = len(blocks)
    est = sc = 0.0
    for w, t in enumerate(blocks):
        fn, fz = local_counts(t, f_nz, f_z, P, w)
        e, s = loss_estimate(t, A_of_rank(w), loss, seed, w, fn, fz, lam)
        est += e
        sc += s
    return est, sc


def slice_groups(grid, k):
    """Ranks sharing b_k, i.e. the mode-k slice communicator."""
    P = math.prod(grid)
    groups = {}
    for w in range(P):
        groups.setdefault(rank_coords(w, grid)[k], []).append(w)
    return [groups[b] for b in sorted(groups)]


class MultiRank:
    """State of a P-rank run and one iteration of Alg. 2 (sync), Alg. 3
    (LocalSGD, reading R16) or Alg. 4 (FedAdam, reading R17), with the
    iteration counter semantics of reading R18."""

    def __init__(self, blocks, grid, A0, loss, mode="sync", beta1=0.9, beta2=0.999, eps=1e-8,
                 lower=None, strategy="stratified", tau=1, meta_rate=1e-3, lam=None):
        self.blocks, self.grid, self.loss, self.mode = blocks, grid, loss, mode
        self.P, self.d = len(blocks), len(A0)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.lower = loss_lower(loss) if lower is None else lower
        self.strategy, self.tau, self.meta_rate, self.lam = strategy, tau, meta_rate, lam
        self.R = A0[0].shape[1]
        self.dims = [a.shape[0] for a in A0]
        if mode == "sync":
            self.st = {"A": [np.array(a, np.float64) for a in A0],
                       "B": [np.zeros_like(a, np.float64) for a in A0],
                       "C": [np.zeros_like(a, np.float64) for a in A0], "t": 0}
        else:
            st = {"A": [], "B": [], "C": [], "t": [0] * self.P, "U": [], "Bs": [], "Cs": [], "ts": [0] * self.P}
            for w, tb in enumerate(blocks):
                Aw = [np.array(A0[k][tb.lo[k]:tb.hi[k]], np.float64) for k in range(self.d)]
                st["A"].append(Aw)
                st["B"].append([np.zeros_like(a) for a in Aw])
                st["C"].append([np.zeros_like(a) for a in Aw])
                st["U"].append([a.copy() for a in Aw])
                st["Bs"].append([np.zeros_like(a) for a in Aw])
                st["Cs"].append([np.zeros_like(a) for a in Aw])
            self.st = st

    def model_for_rank(self, w):
        """Global-shaped factors as rank w sees them (its replica in async modes)."""
        if self.mode == "sync":
            return self.st["A"]
        tb = self.blocks[w]
        full = [np.zeros((self.dims[k], self.R)) for k in range(self.d)]
        for k in range(self.d):
            full[k][tb.lo[k]:tb.hi[k]] = self.st["A"][w][k]
        return full

    def block_rows(self, w, k):
        tb = self.blocks[w]
        if self.mode == "sync":
            return self.st["A"][k][tb.lo[k]:tb.hi[k]]
        return self.st["A"][w][k]

    def _adam_list(self, As, Gs, Bs, Cs, t, rate):
        for k in range(self.d):
            adam(As[k].reshape(-1), np.ascontiguousarray(Gs[k], np.float64).reshape(-1),
                 Bs[k].reshape(-1), Cs[k].reshape(-1), t, rate, self.beta1, self.beta2, self.eps, self.lower)

    def async_sync(self):
        """Alg. 3 lines 2-4 / Alg. 4 lines 3-6 over every mode's slice groups."""
        st = self.st
        for k in range(self.d):
            for grp in slice_groups(self.grid, k):
                if self.mode == "async":      # average over the g_k replicas
                    avg = sum(st["A"][w][k] for w in grp) / len(grp)
                    for w in grp:
                        st["A"][w][k][...] = avg
                else:                         # D = U - M, AllReduce(D) (sum), server Adam on U, M <- U
                    S = sum(st["U"][w][k] - st["A"][w][k] for w in grp)
                    for w in grp:
                        adam(st["U"][w][k].reshape(-1), np.ascontiguousarray(S, np.float64).reshape(-1),
                             st["Bs"][w][k].reshape(-1), st["Cs"][w][k].reshape(-1), st["ts"][w] + 1,
                             self.meta_rate, self.beta1, self.beta2, self.eps, self.lower)
                        st["A"][w][k][...] = st["U"][w][k]
        if self.mode == "fedadam":
            for w in range(self.P):
                st["ts"][w] += 1

    def iteration(self, it, seed, s_nz, s_z, rate):
        """One mini-batch iteration with Philox iteration word `it`."""
        st = self.st
        if self.mode == "sync":
            G, _, _ = sync_gradient(self.blocks, st["A"], self.loss, seed, it, s_nz, s_z, self.strategy, self.lam)
            st["t"] += 1
            self._adam_list(st["A"], G, st["B"], st["C"], st["t"], rate)
            return
        if (it + 1) % self.tau == 0:
            self.async_sync()
        for w, tb in enumerate(self.blocks):
            pw, qw = local_counts(tb, s_nz, s_z, self.P, w)
            Gw, _, _ = sampled_grad(tb, self.model_for_rank(w), self.loss, seed, w, it, pw, qw,
                                    self.strategy, self.lam, with_scale=False)
            st["t"][w] += 1
            self._adam_list(st["A"][w], Gw, st["B"][w], st["C"][w], st["t"][w], rate)

    def estimate(self, fseed, f_nz, f_z):
        return sync_loss_estimate(self.blocks, self.model_for_rank, self.loss, fseed, f_nz, f_z, self.lam)


def fit(blocks, grid, A0, loss, *, epochs=10, iters=100, max_fails=3, rate=1e-3, decay=0.1,
        beta1=0.9, beta2=0.999, eps=1e-8, lower=None, s_nz=1000, s_z=1000, f_nz=1000,
        f_z=1000, seed=1, fseed=2, strategy="stratified", mode="sync", tau=1,
        meta_rate=None, lam=None, trace=None):
    """Epoch loop with annealing (reading R20) around Alg. 2 / 3 / 4.

    Returns (final factors (global list for sync, per-rank global-shaped lists
    otherwise), list of per-epoch (est_loss, rate, accepted), best estimate)."""
    import copy
    run = MultiRank(blocks, grid, A0, loss, mode, beta1, beta2, eps, lower, strategy, tau,
                    rate if meta_rate is None else meta_rate, lam)
    best = run.estimate(fseed, f_nz, f_z)[0]
    ckpt = copy.deepcopy(run.st)
    it = 0
    fails = 0
    hist = []
    for e in range(epochs):
        for _ in range(iters):
            run.iteration(it, seed, s_nz, s_z, rate)
            it += 1
        est = run.estimate(fseed, f_nz, f_z)[0]
        if est < best:
            best = est
            ckpt = copy.deepcopy(run.st)
            hist.append((est, rate, True))
        else:
            run.st = copy.deepcopy(ckpt)
            hist.append((est, rate, False))
            rate *= decay
            fails += 1
        if trace:
            trace(e, it, est, rate)
        if fails >= max_fails:
            break
    if mode == "sync":
        return run.st["A"], hist, best
    return [run.model_for_rank(w) for w in range(len(blocks))], hist, best
