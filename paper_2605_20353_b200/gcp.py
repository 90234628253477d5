"""Thin ctypes binding of include/gcp.h (argument marshalling only).

Every function here has the name of the C entry point it wraps and does no
arithmetic of the method: all of it runs in libgcp.so's sm_100a kernels.  If
libgcp.so is missing or cannot be loaded, importing this module raises -- there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / os.environ.get("GCP_LIB", "libgcp.so")

GCP_OK = 0
STATUS = {0: "GCP_OK", 1: "GCP_E_ARG", 2: "GCP_E_RANGE", 3: "GCP_E_DUP", 4: "GCP_E_NO_NONZEROS",
          5: "GCP_E_NO_ZEROS", 6: "GCP_E_REJECT_CAP", 7: "GCP_E_STATE", 8: "GCP_E_OOM", 9: "GCP_E_CUDA",
          10: "GCP_E_NCCL"}
LOSS = {"gaussian": 0, "poisson": 1, "bernoulli": 2}
STRATEGY = {"stratified": 0, "semi": 1}
PRECISION = {"fp32": 0, "fp64": 1}
DIST_MODE = {"sync": 0, "async": 1, "fedadam": 2, "twosided": 3}
PROF = {"grad": 0, "adam": 1, "loss": 2, "comm": 3, "other": 4}

# every symbol include/gcp.h declares (checked by tests/test_abi.py)
SYMBOLS = ["gcp_create", "gcp_destroy", "gcp_last_error", "gcp_grid_plan", "gcp_nccl_unique_id",
           "gcp_dist_init", "gcp_dist_set_async", "gcp_tensor_create", "gcp_tensor_info",
           "gcp_tensor_export_sorted", "gcp_tensor_contains", "gcp_model_init", "gcp_model_set",
           "gcp_model_get", "gcp_sample", "gcp_sample_export", "gcp_loss_grad", "gcp_grad_get",
           "gcp_adam_step", "gcp_loss_estimate", "gcp_fit_begin", "gcp_fit_epoch", "gcp_fit",
           "gcp_counters", "gcp_profile_enable", "gcp_profile_get", "gcp_set_membership",
           "gcp_dist_features", "gcp_layout", "gcp_debug_nonzero_j", "gcp_debug_philox"]
MEMBERSHIP = {"hash": 0, "sorted": 1}


class GcpError(RuntimeError):
    def __init__(self, code, where, msg):
        self.code = code
        self.name = STATUS.get(code, str(code))
        super().__init__(f"{where}: {self.name}: {msg}")


class AdamParams(C.Structure):
    _fields_ = [("rate", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("lower", C.c_double)]


class FitParams(C.Structure):
    _fields_ = [("epochs", C.c_int), ("iters_per_epoch", C.c_int), ("max_fails", C.c_int),
                ("decay", C.c_double), ("s_nz", C.c_int64), ("s_z", C.c_int64),
                ("f_nz", C.c_int64), ("f_z", C.c_int64), ("strategy", C.c_int), ("loss", C.c_int),
                ("seed", C.c_uint64), ("fseed", C.c_uint64), ("adam", AdamParams),
                ("tau", C.c_int64), ("meta_rate", C.c_double)]


TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double)


def load():
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} is missing: run `python paper_2605_20353_b200/build.py` "
                          "(there is no CPU fallback)")
    L = C.CDLL(str(_LIB_PATH))
    vp, i64, i64p, dp, ip = C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_int)
    sig = {
        "gcp_create": [C.POINTER(vp), C.c_int, vp, C.c_int],
        "gcp_grid_plan": [C.c_int, C.c_int, i64p, ip, i64p, i64p],
        "gcp_nccl_unique_id": [vp],
        "gcp_dist_init": [vp, C.c_int, C.c_int, vp, ip, C.c_int, C.c_int],
        "gcp_dist_set_async": [vp, i64, C.POINTER(AdamParams)],
        "gcp_tensor_create": [vp, C.c_int, i64p, i64, i64p, dp],
        "gcp_tensor_info": [vp, i64p, i64p, i64p, dp, i64p],
        "gcp_tensor_export_sorted": [vp, i64, i64, i64p, dp],
        "gcp_tensor_contains": [vp, i64, i64p, C.POINTER(C.c_int8)],
        "gcp_model_init": [vp, C.c_int, C.c_uint64],
        "gcp_model_set": [vp, C.c_int, dp, dp],
        "gcp_model_get": [vp, C.c_int, dp],
        "gcp_sample": [vp, C.c_int, i64, i64, C.c_uint64],
        "gcp_sample_export": [vp, C.c_int, i64, i64, i64p, i64p, dp, C.POINTER(C.c_int32)],
        "gcp_loss_grad": [vp, C.c_int, dp],
        "gcp_grad_get": [vp, C.c_int, dp],
        "gcp_adam_step": [vp, C.POINTER(AdamParams)],
        "gcp_loss_estimate": [vp, C.c_int, i64, i64, C.c_uint64, dp],
        "gcp_fit_begin": [vp, C.POINTER(FitParams), dp],
        "gcp_fit_epoch": [vp, dp, ip, ip],
        "gcp_fit": [vp, C.POINTER(FitParams), TRACE_FN, vp, dp],
        "gcp_counters": [vp, C.POINTER(C.c_uint32), i64p, i64p],
        "gcp_dist_features": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "gcp_layout": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "gcp_debug_nonzero_j": [vp, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int64, C.c_int64, C.c_int64, i64p],
        "gcp_debug_philox": [vp, C.c_int64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)],
        "gcp_profile_enable": [vp, C.c_int],
        "gcp_profile_get": [vp, C.c_int, dp, i64p, C.c_int],
        "gcp_set_membership": [vp, C.c_int],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.gcp_destroy.argtypes = [vp]
    L.gcp_destroy.restype = None
    L.gcp_last_error.argtypes = []
    L.gcp_last_error.restype = C.c_char_p
    return L


lib = load()


def _chk(st, where):
    if st != GCP_OK:
        raise GcpError(st, where, lib.gcp_last_error().decode())


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def adam_params(rate=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, lower=math.nan):
    return AdamParams(rate, beta1, beta2, eps, lower)


def gcp_grid_plan(P, dims):
    d = len(dims)
    dims_a = _i64(dims)
    grid = (C.c_int * d)()
    lo = np.zeros(P * d, np.int64)
    hi = np.zeros(P * d, np.int64)
    _chk(lib.gcp_grid_plan(P, d, _ptr(dims_a, C.c_int64), grid, _ptr(lo, C.c_int64), _ptr(hi, C.c_int64)),
         "gcp_grid_plan")
    return tuple(grid), lo.reshape(P, d), hi.reshape(P, d)


def gcp_nccl_unique_id():
    buf = (C.c_char * 128)()
    _chk(lib.gcp_nccl_unique_id(buf), "gcp_nccl_unique_id")
    return bytes(buf)


class Context:
    """One gcp_ctx (one rank / one GPU).  Methods are the C entry points minus
    the `gcp_` prefix, with numpy in place of raw pointers."""

    def __init__(self, device=0, stream=None, precision="fp32"):
        h = C.c_void_p()
        s = None if stream is None else C.c_void_p(int(stream))
        _chk(lib.gcp_create(C.byref(h), int(device), s, PRECISION[precision]), "gcp_create")
        self.h = h
        self.precision = precision
        self.d = None
        self.R = None

    def close(self):
        if getattr(self, "h", None):
            lib.gcp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- distribution
    def dist_init(self, nranks, rank, unique_id=None, grid=None, mode="sync"):
        idbuf = None if unique_id is None else C.create_string_buffer(bytes(unique_id), 128)
        g = None if grid is None else (C.c_int * len(grid))(*grid)
        _chk(lib.gcp_dist_init(self.h, nranks, rank, idbuf, g, 0 if grid is None else len(grid),
                               DIST_MODE[mode]), "gcp_dist_init")

    def dist_set_async(self, tau, server=None):
        _chk(lib.gcp_dist_set_async(self.h, int(tau), None if server is None else C.byref(server)),
             "gcp_dist_set_async")

    # ---- tensor
    def set_membership(self, m):
        _chk(lib.gcp_set_membership(self.h, MEMBERSHIP[m]), "gcp_set_membership")

    def tensor_create(self, dims, subs, vals):
        dims_a = _i64(dims)
        subs_a = _i64(subs).reshape(-1)
        vals_a = _f64(vals)
        self.d = len(dims)
        self.dims = [int(x) for x in dims]
        _chk(lib.gcp_tensor_create(self.h, len(dims), _ptr(dims_a, C.c_int64), len(vals_a),
                                   _ptr(subs_a, C.c_int64), _ptr(vals_a, C.c_double)), "gcp_tensor_create")

    def tensor_create_ptr(self, dims, nnz, subs_ptr, vals_ptr):
        """Same as tensor_create, from raw (e.g. pinned torch) host pointers."""
        dims_a = _i64(dims)
        self.d = len(dims)
        self.dims = [int(x) for x in dims]
        _chk(lib.gcp_tensor_create(self.h, len(dims), _ptr(dims_a, C.c_int64), int(nnz),
                                   C.cast(C.c_void_p(subs_ptr), C.POINTER(C.c_int64)),
                                   C.cast(C.c_void_p(vals_ptr), C.POINTER(C.c_double))), "gcp_tensor_create")

    def tensor_info(self):
        n, ng = C.c_int64(), C.c_int64()
        lo = np.zeros(self.d, np.int64)
        hi = np.zeros(self.d, np.int64)
        M = C.c_double()
        _chk(lib.gcp_tensor_info(self.h, C.byref(n), _ptr(lo, C.c_int64), _ptr(hi, C.c_int64), C.byref(M),
                                 C.byref(ng)), "gcp_tensor_info")
        return dict(nnz=n.value, lo=lo, hi=hi, M=M.value, nnz_global=ng.value)

    def tensor_export_sorted(self, first, count):
        s = np.zeros((count, self.d), np.int64)
        v = np.zeros(count, np.float64)
        _chk(lib.gcp_tensor_export_sorted(self.h, first, count, _ptr(s, C.c_int64), _ptr(v, C.c_double)),
             "gcp_tensor_export_sorted")
        return s, v

    def tensor_contains(self, coords):
        c = _i64(coords).reshape(-1, self.d)
        out = np.zeros(len(c), np.int8)
        _chk(lib.gcp_tensor_contains(self.h, len(c), _ptr(c, C.c_int64), _ptr(out, C.c_int8)),
             "gcp_tensor_contains")
        return out.astype(bool)

    # ---- model
    def model_init(self, R, seed):
        self.R = int(R)
        _chk(lib.gcp_model_init(self.h, int(R), C.c_uint64(seed)), "gcp_model_init")

    def _block_rows(self, k):
        info = self.tensor_info()
        return int(info["hi"][k] - info["lo"][k])

    def model_set(self, k, rows, lam=None):
        r = _f64(rows)
        la = None if lam is None else _f64(lam)
        _chk(lib.gcp_model_set(self.h, k, _ptr(r, C.c_double), _ptr(la, C.c_double)), "gcp_model_set")

    def model_get(self, k):
        out = np.zeros((self._block_rows(k), self.R), np.float64)
        _chk(lib.gcp_model_get(self.h, k, _ptr(out, C.c_double)), "gcp_model_get")
        return out

    # ---- sampling / gradient
    def sample(self, strategy, s_nz, s_z, seed):
        _chk(lib.gcp_sample(self.h, STRATEGY[strategy], int(s_nz), int(s_z), C.c_uint64(seed)), "gcp_sample")

    def sample_export(self, stratum, first, count):
        s = np.zeros((count, self.d), np.int64)
        j = np.zeros(count, np.int64)
        w = np.zeros(count, np.float64)
        a = np.zeros(count, np.int32)
        _chk(lib.gcp_sample_export(self.h, stratum, first, count, _ptr(s, C.c_int64), _ptr(j, C.c_int64),
                                   _ptr(w, C.c_double), _ptr(a, C.c_int32)), "gcp_sample_export")
        return s, j, w, a

    def loss_grad(self, loss, want_loss=False):
        out = C.c_double()
        _chk(lib.gcp_loss_grad(self.h, LOSS[loss], C.byref(out) if want_loss else None), "gcp_loss_grad")
        return out.value if want_loss else None

    def grad_get(self, k):
        out = np.zeros((self._block_rows(k), self.R), np.float64)
        _chk(lib.gcp_grad_get(self.h, k, _ptr(out, C.c_double)), "gcp_grad_get")
        return out

    def adam_step(self, params=None):
        p = params if params is not None else adam_params()
        _chk(lib.gcp_adam_step(self.h, C.byref(p)), "gcp_adam_step")

    def loss_estimate(self, loss, f_nz, f_z, seed):
        out = C.c_double()
        _chk(lib.gcp_loss_estimate(self.h, LOSS[loss], int(f_nz), int(f_z), C.c_uint64(seed), C.byref(out)),
             "gcp_loss_estimate")
        return out.value

    # ---- fit
    @staticmethod
    def fit_params(epochs=10, iters_per_epoch=100, max_fails=3, decay=0.1, s_nz=1000, s_z=1000, f_nz=1000,
                   f_z=1000, strategy="stratified", loss="poisson", seed=1, fseed=2, rate=1e-3, beta1=0.9,
                   beta2=0.999, eps=1e-8, lower=math.nan, tau=0, meta_rate=0.0):
        return FitParams(epochs, iters_per_epoch, max_fails, decay, s_nz, s_z, f_nz, f_z, STRATEGY[strategy],
                         LOSS[loss], seed, fseed, AdamParams(rate, beta1, beta2, eps, lower), tau, meta_rate)

    def fit_begin(self, params):
        out = C.c_double()
        _chk(lib.gcp_fit_begin(self.h, C.byref(params), C.byref(out)), "gcp_fit_begin")
        return out.value

    def fit_epoch(self):
        est, acc, done = C.c_double(), C.c_int(), C.c_int()
        _chk(lib.gcp_fit_epoch(self.h, C.byref(est), C.byref(acc), C.byref(done)), "gcp_fit_epoch")
        return est.value, bool(acc.value), bool(done.value)

    def fit(self, params, trace=None):
        rows = []

        def _cb(user, epoch, it, est, rate, el):
            rows.append((epoch, it, est, rate, el))
            if trace:
                trace(epoch, it, est, rate, el)

        cb = TRACE_FN(_cb)
        out = C.c_double()
        _chk(lib.gcp_fit(self.h, C.byref(params), cb, None, C.byref(out)), "gcp_fit")
        return out.value, rows

    # ---- instrumentation
    def counters(self):
        it, t, n = C.c_uint32(), C.c_int64(), C.c_int64()
        _chk(lib.gcp_counters(self.h, C.byref(it), C.byref(t), C.byref(n)), "gcp_counters")
        return dict(it=it.value, t=t.value, launches=n.value)

    def dist_features(self):
        f, m = C.c_int(), C.c_int()
        _chk(lib.gcp_dist_features(self.h, C.byref(f), C.byref(m)), "gcp_dist_features")
        return dict(fused=bool(f.value), multimem=bool(m.value))

    def layout(self):
        a, o, f = C.c_int(), C.c_int(), C.c_int()
        _chk(lib.gcp_layout(self.h, C.byref(a), C.byref(o), C.byref(f)), "gcp_layout")
        return dict(ag_interleaved=bool(a.value), slot_order=bool(o.value), filter=bool(f.value))

    def debug_nonzero_j(self, seed, rank, it, N, first, count):
        out = np.zeros(count, np.int64)
        _chk(lib.gcp_debug_nonzero_j(self.h, seed, rank, it, N, first, count, _ptr(out, C.c_int64)),
             "gcp_debug_nonzero_j")
        return out

    def debug_philox(self, ctr_key):
        """(n, 6) uint32 (counter, key) -> (ours (n, 4), curand (n, 4))."""
        a = np.ascontiguousarray(ctr_key, dtype=np.uint32).reshape(-1, 6)
        out = np.zeros((a.shape[0], 8), np.uint32)
        _chk(lib.gcp_debug_philox(self.h, a.shape[0], _ptr(a, C.c_uint32), _ptr(out, C.c_uint32)), "gcp_debug_philox")
        return out[:, :4], out[:, 4:]

    def profile_enable(self, on=True):
        _chk(lib.gcp_profile_enable(self.h, int(on)), "gcp_profile_enable")

    def profile_get(self, which, reset=False):
        ms, n = C.c_double(), C.c_int64()
        _chk(lib.gcp_profile_get(self.h, PROF[which], C.byref(ms), C.byref(n), int(reset)), "gcp_profile_get")
        return ms.value, n.value
