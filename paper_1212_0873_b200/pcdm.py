"""Thin ctypes binding of libpcdm.so (include/pcdm.h), same names as the C ABI.

Argument marshalling only: every step of the PCDM1 path runs in the library's
CUDA kernels.  Arrays may be torch tensors (CUDA or CPU) or numpy arrays; they
must already have the ABI's dtype (int64 colptr, int32 rowidx, float32
val/b/x/L/r) and be contiguous.  ``stream=None`` means torch's current CUDA
stream.  There is no CPU fallback: if libpcdm.so is missing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpcdm.so")

PCDM_OK, PCDM_EINVAL, PCDM_ENOMEM, PCDM_ECUDA, PCDM_EDIVERGED, PCDM_ESAMPLER = range(6)
VARIANTS = {"auto": 0, "grid": 1, "smem": 2, "block": 3, "packed": 4, "batched": 5}
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "EDIVERGED", 5: "ESAMPLER"}

EXPORTS = ["pcdm_create", "pcdm_destroy", "pcdm_last_error", "pcdm_omega", "pcdm_beta", "pcdm_run",
           "pcdm_run_ex", "pcdm_objective", "pcdm_last_run_stats", "pcdm_sample", "pcdm_col_norms",
           "pcdm_row_counts", "pcdm_residual", "pcdm_philox", "pcdm_philox_check_curand",
           "pcdm_run_sampling", "pcdm_beta_sampling", "pcdm_sample_sampling", "pcdm_run_async",
           "pcdm_create_logistic"]
SAMPLING_KINDS = {"nice": 0, "independent": 1, "binomial": 2, "du": 3}


class PCDMError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), message))
        self.status = status
        self.message = message


class RunStats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int64), ("nonzero_deltas", ctypes.c_int64),
                ("sampler_max_rounds", ctypes.c_int64), ("refreshes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("variant", ctypes.c_int32),
                ("grid_ctas", ctypes.c_int32), ("threads_per_cta", ctypes.c_int32),
                ("lanes_per_column", ctypes.c_int32), ("chunk_iters", ctypes.c_int64),
                ("iter_launches", ctypes.c_int64), ("iter_kernel_ms", ctypes.c_double),
                ("sampler_ms", ctypes.c_double), ("setup_ms", ctypes.c_double),
                ("hot_rows", ctypes.c_int64), ("host_h2d_bytes", ctypes.c_int64),
                ("host_d2h_bytes", ctypes.c_int64), ("screen_misses", ctypes.c_int64),
                ("screen_scans", ctypes.c_int64), ("screen_spec", ctypes.c_int64),
                ("screen_flagged", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class _CSampling(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("tau", ctypes.c_int64),
                ("p_b", ctypes.c_double), ("q", ctypes.c_void_p)]


class Sampling:
    """A doubly uniform sampling for pcdm_run_sampling (include/pcdm.h): kind in
    SAMPLING_KINDS, tau slots, p_b (binomial), q[0..tau] (du)."""

    def __init__(self, kind="nice", tau=1, p_b=1.0, q=None):
        if kind not in SAMPLING_KINDS:
            raise ValueError("unknown sampling kind %r" % kind)
        self.kind, self.tau, self.p_b = kind, int(tau), float(p_b)
        self.q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)

    def c(self):
        return _CSampling(SAMPLING_KINDS[self.kind], 0, self.tau, self.p_b,
                          None if self.q is None else self.q.ctypes.data)


_lib = None


def load():
    """Load libpcdm.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError("libpcdm.so not built: run `python -m paper_1212_0873_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, i64, u64, i32, f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double
    st = ctypes.c_int
    sig = {
        "pcdm_create": ([i64, i64, i64, P, P, P, P, f64, P, ctypes.POINTER(P)], st),
        "pcdm_destroy": ([P], None),
        "pcdm_last_error": ([], ctypes.c_char_p),
        "pcdm_omega": ([P, ctypes.POINTER(i64)], st),
        "pcdm_beta": ([P, i64, ctypes.POINTER(f64)], st),
        "pcdm_run": ([P, P, i64, i64, u64, P], st),
        "pcdm_run_ex": ([P, P, i64, i64, u64, i64, i64, f64, i32, P], st),
        "pcdm_objective": ([P, P, ctypes.POINTER(f64), P], st),
        "pcdm_last_run_stats": ([P, ctypes.POINTER(RunStats)], st),
        "pcdm_sample": ([i64, i64, u64, i64, i64, P, P], st),
        "pcdm_col_norms": ([P, P, P], st),
        "pcdm_row_counts": ([P, P, P], st),
        "pcdm_residual": ([P, P, P], st),
        "pcdm_philox": ([i64, P, P, P, P], st),
        "pcdm_philox_check_curand": ([i64, u64, ctypes.POINTER(i64), P], st),
        "pcdm_run_sampling": ([P, P, ctypes.POINTER(_CSampling), i64, u64, i64, i64, f64, i32, P], st),
        "pcdm_run_async": ([P, P, i64, i64, f64, i64, u64, u64, P], st),
        "pcdm_create_logistic": ([i64, i64, i64, P, P, P, P, f64, P, ctypes.POINTER(P)], st),
        "pcdm_beta_sampling": ([P, ctypes.POINTER(_CSampling), ctypes.POINTER(f64)], st),
        "pcdm_sample_sampling": ([i64, ctypes.POINTER(_CSampling), u64, i64, i64, P, P], st),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(status: int):
    if status != PCDM_OK:
        raise PCDMError(status, load().pcdm_last_error().decode())


_DT = {"i64": ("int64", np.int64), "i32": ("int32", np.int32), "u32": ("uint32", np.uint32),
       "f32": ("float32", np.float32)}


def _ptr(a, kind: str):
    """data pointer of a contiguous torch tensor / numpy array of the ABI dtype."""
    tname, npd = _DT[kind]
    if isinstance(a, np.ndarray):
        if a.dtype != npd or not a.flags["C_CONTIGUOUS"]:
            raise TypeError("expected contiguous %s numpy array" % tname)
        return ctypes.c_void_p(a.ctypes.data)
    import torch
    if not isinstance(a, torch.Tensor):
        raise TypeError("expected torch.Tensor or numpy.ndarray")
    if a.dtype != getattr(torch, tname) or not a.is_contiguous():
        raise TypeError("expected contiguous torch.%s tensor, got %s" % (tname, a.dtype))
    return ctypes.c_void_p(a.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(0)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def pcdm_last_error() -> str:
    return load().pcdm_last_error().decode()


def pcdm_create(m, n, colptr, rowidx, val, b, lam, stream=None):
    nnz = int(rowidx.shape[0]) if hasattr(rowidx, "shape") else len(rowidx)
    h = ctypes.c_void_p()
    _check(load().pcdm_create(int(m), int(n), nnz, _ptr(colptr, "i64"), _ptr(rowidx, "i32"),
                              _ptr(val, "f32"), _ptr(b, "f32"), float(lam), _stream(stream),
                              ctypes.byref(h)))
    return h


def pcdm_create_logistic(m, n, colptr, rowidx, val, y, lam, stream=None):
    nnz = int(rowidx.shape[0]) if hasattr(rowidx, "shape") else len(rowidx)
    h = ctypes.c_void_p()
    _check(load().pcdm_create_logistic(int(m), int(n), nnz, _ptr(colptr, "i64"), _ptr(rowidx, "i32"),
                                       _ptr(val, "f32"), _ptr(y, "f32"), float(lam), _stream(stream),
                                       ctypes.byref(h)))
    return h


def pcdm_destroy(h):
    if h:
        load().pcdm_destroy(h)


def pcdm_omega(h) -> int:
    v = ctypes.c_int64()
    _check(load().pcdm_omega(h, ctypes.byref(v)))
    return v.value


def pcdm_beta(h, tau) -> float:
    v = ctypes.c_double()
    _check(load().pcdm_beta(h, int(tau), ctypes.byref(v)))
    return v.value


def pcdm_run(h, x, tau, iters, seed, stream=None):
    _check(load().pcdm_run(h, _ptr(x, "f32"), int(tau), int(iters), int(seed), _stream(stream)))


def pcdm_run_ex(h, x, tau, iters, seed, first_iter=0, refresh_every=0, beta_override=0.0,
                variant="auto", stream=None):
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    _check(load().pcdm_run_ex(h, _ptr(x, "f32"), int(tau), int(iters), int(seed), int(first_iter),
                              int(refresh_every), float(beta_override), v, _stream(stream)))


def pcdm_run_sampling(h, x, sampling: Sampling, iters, seed, first_iter=0, refresh_every=0, beta_override=0.0,
                      variant="auto", stream=None):
    v = VARIANTS[variant] if isinstance(variant, str) else int(variant)
    cs = sampling.c()
    _check(load().pcdm_run_sampling(h, _ptr(x, "f32"), ctypes.byref(cs), int(iters), int(seed), int(first_iter),
                                    int(refresh_every), float(beta_override), v, _stream(stream)))


def pcdm_run_async(h, x, updates, tau_beta=0, beta_override=0.0, refresh_every=0, first_update=0, seed=0,
                   stream=None):
    _check(load().pcdm_run_async(h, _ptr(x, "f32"), int(updates), int(tau_beta), float(beta_override),
                                 int(refresh_every), int(first_update), int(seed), _stream(stream)))


def pcdm_beta_sampling(h, sampling: Sampling) -> float:
    v = ctypes.c_double()
    cs = sampling.c()
    _check(load().pcdm_beta_sampling(h, ctypes.byref(cs), ctypes.byref(v)))
    return v.value


def pcdm_sample_sampling(n, sampling: Sampling, seed, first_iter, count, out, stream=None):
    cs = sampling.c()
    _check(load().pcdm_sample_sampling(int(n), ctypes.byref(cs), int(seed), int(first_iter), int(count),
                                       _ptr(out, "i32"), _stream(stream)))
    return out


def pcdm_objective(h, x, stream=None) -> float:
    F = ctypes.c_double()
    _check(load().pcdm_objective(h, _ptr(x, "f32"), ctypes.byref(F), _stream(stream)))
    return F.value


def pcdm_last_run_stats(h) -> dict:
    s = RunStats()
    _check(load().pcdm_last_run_stats(h, ctypes.byref(s)))
    return s.as_dict()


def pcdm_sample(n, tau, seed, first_iter, count, out, stream=None):
    _check(load().pcdm_sample(int(n), int(tau), int(seed), int(first_iter), int(count),
                              _ptr(out, "i32"), _stream(stream)))
    return out


def pcdm_col_norms(h, out, stream=None):
    _check(load().pcdm_col_norms(h, _ptr(out, "f32"), _stream(stream)))
    return out


def pcdm_row_counts(h, out, stream=None):
    _check(load().pcdm_row_counts(h, _ptr(out, "i32"), _stream(stream)))
    return out


def pcdm_residual(h, out, stream=None):
    _check(load().pcdm_residual(h, _ptr(out, "f32"), _stream(stream)))
    return out


def pcdm_philox(ctr, key, out, stream=None):
    count = int(out.shape[0]) // 4
    _check(load().pcdm_philox(count, _ptr(ctr, "u32"), _ptr(key, "u32"), _ptr(out, "u32"),
                              _stream(stream)))
    return out


def pcdm_philox_check_curand(count, seed, stream=None) -> int:
    v = ctypes.c_int64()
    _check(load().pcdm_philox_check_curand(int(count), int(seed), ctypes.byref(v), _stream(stream)))
    return v.value


class Problem:
    """Owning wrapper around a pcdm_problem handle (destroyed on close / GC)."""

    def __init__(self, m, n, colptr, rowidx, val, b, lam, stream=None, loss="lasso"):
        """loss "lasso": b is the target; loss "logistic": b holds the labels y (+-1)."""
        self.m, self.n, self.nnz, self.lam = int(m), int(n), int(rowidx.shape[0]), float(lam)
        self.loss = loss
        if loss == "lasso":
            self.handle = pcdm_create(m, n, colptr, rowidx, val, b, lam, stream)
        elif loss == "logistic":
            self.handle = pcdm_create_logistic(m, n, colptr, rowidx, val, b, lam, stream)
        else:
            raise ValueError("loss must be 'lasso' or 'logistic'")

    @classmethod
    def from_instance(cls, inst, stream=None):
        return cls(inst.m, inst.n, inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, stream)

    def close(self):
        if getattr(self, "handle", None):
            try:
                pcdm_destroy(self.handle)
            except Exception:  # interpreter shutdown: module globals already gone
                pass
            self.handle = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def omega(self):
        return pcdm_omega(self.handle)

    def beta(self, tau):
        return pcdm_beta(self.handle, tau)

    def run(self, x, tau, iters, seed=0, first_iter=0, refresh_every=0, beta_override=0.0,
            variant="auto", stream=None, sampling: Sampling = None):
        """PCDM1 iterations; tau-nice unless `sampling` is given (then tau is ignored)."""
        if sampling is None:
            pcdm_run_ex(self.handle, x, tau, iters, seed, first_iter, refresh_every, beta_override,
                        variant, stream)
        else:
            pcdm_run_sampling(self.handle, x, sampling, iters, seed, first_iter, refresh_every, beta_override,
                              variant, stream)
        return x

    def run_async(self, x, updates, tau_beta=0, beta_override=0.0, refresh_every=0, first_update=0, seed=0,
                  stream=None):
        """Asynchronous variant (NEXT-4): `updates` coordinate updates, no barriers."""
        pcdm_run_async(self.handle, x, updates, tau_beta, beta_override, refresh_every, first_update, seed, stream)
        return x

    def beta_sampling(self, sampling: Sampling):
        return pcdm_beta_sampling(self.handle, sampling)

    def objective(self, x, stream=None):
        return pcdm_objective(self.handle, x, stream)

    def stats(self):
        return pcdm_last_run_stats(self.handle)

    def col_norms(self, out, stream=None):
        return pcdm_col_norms(self.handle, out, stream)

    def row_counts(self, out, stream=None):
        return pcdm_row_counts(self.handle, out, stream)

    def residual(self, out, stream=None):
        return pcdm_residual(self.handle, out, stream)
