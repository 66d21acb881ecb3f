"""PCDM1/LASSO serial CPU oracle (ctypes wrapper around oracle/pcdm_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1212_0873_b200`` never imports it and
shares no code with it ("Oracle").

Every function follows the paper step by step in fp64; the C source cites the
PAPER.md lines for each step.  Array arguments are numpy arrays on the host.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pcdm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 (no fast-math, no OpenMP, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_POSIX_C_SOURCE=199309L", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB)
    P = ctypes.c_void_p
    i64, u64, u32, f64, i32 = (ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32,
                               ctypes.c_double, ctypes.c_int)
    lib.or_philox4x32_10.argtypes = [P, P, P]
    lib.or_philox4x32_10.restype = None
    lib.or_draw.argtypes = [u64, u32, u32, u32, u32, u64, ctypes.POINTER(ctypes.c_uint64)]
    lib.or_draw.restype = i32
    lib.or_sample.argtypes = [u64, i64, i64, i64, P, P]
    lib.or_sample.restype = i32
    lib.or_row_counts.argtypes = [i64, P, P]
    lib.or_row_counts.restype = None
    lib.or_omega.argtypes = [i64, i64, P]
    lib.or_omega.restype = i64
    lib.or_col_norms.argtypes = [i64, P, P, P]
    lib.or_col_norms.restype = None
    lib.or_beta.argtypes = [i64, i64, i64]
    lib.or_beta.restype = f64
    lib.or_prox.argtypes = [f64, f64, f64, f64]
    lib.or_prox.restype = f64
    lib.or_residual.argtypes = [i64, i64, P, P, P, P, P, P]
    lib.or_residual.restype = None
    lib.or_objective.argtypes = [i64, i64, P, P, P, P, f64, P]
    lib.or_objective.restype = f64
    lib.or_refresh_period.argtypes = [i64, i64, i64]
    lib.or_refresh_period.restype = i64
    lib.or_run.argtypes = [i64, i64, P, P, P, P, f64, P, f64, P, i64, i64, u64, i64, i64,
                           P, P, ctypes.POINTER(ctypes.c_double)]
    lib.or_run.restype = i32
    lib.or_sample_kind.argtypes = [i32, u64, i64, i64, i64, f64, P, P]
    lib.or_sample_kind.restype = i32
    lib.or_moments.argtypes = [i32, i64, i64, f64, P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    lib.or_moments.restype = i32
    lib.or_beta_du.argtypes = [i64, i64, f64, f64]
    lib.or_beta_du.restype = f64
    lib.or_run_kind.argtypes = [i64, i64, P, P, P, P, f64, P, f64, P, i32, i64, f64, P, i64, u64, i64, i64,
                                P, P, ctypes.POINTER(ctypes.c_double)]
    lib.or_run_kind.restype = i32
    lib.or_margins.argtypes = [i64, i64, P, P, P, P, P, P]
    lib.or_margins.restype = None
    lib.or_logistic_objective.argtypes = [i64, i64, P, P, P, P, f64, P]
    lib.or_logistic_objective.restype = f64
    lib.or_logistic_grad_i.argtypes = [P, P, P, P, P, i64]
    lib.or_logistic_grad_i.restype = f64
    lib.or_logistic_L.argtypes = [i64, P, P, P]
    lib.or_logistic_L.restype = None
    lib.or_logistic_step.argtypes = [f64, f64, f64, f64]
    lib.or_logistic_step.restype = f64
    lib.or_logistic_run.argtypes = [i64, i64, P, P, P, P, f64, P, f64, P, i32, i64, f64, P, i64, u64, i64, i64,
                                    P, ctypes.POINTER(ctypes.c_double)]
    lib.or_logistic_run.restype = i32
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _csc(colptr, rowidx, val):
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    val = np.ascontiguousarray(val, dtype=np.float32)
    return colptr, rowidx, val


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def draw(seed: int, k: int, rho: int, j: int, tag: int, n: int):
    """One Lemire-mapped draw; returns the value in [0,n) or None if rejected."""
    v = ctypes.c_uint64(0)
    ok = _load().or_draw(seed, k, rho, j, tag, n, ctypes.byref(v))
    return int(v.value) if ok else None


def sample(seed: int, k: int, tau: int, n: int, workspace: np.ndarray = None) -> np.ndarray:
    """O5: slot array of S_k (tau distinct indices in [0, n)).
    workspace: optional zeroed uint8[n] scratch (or_sample's `taken`, left zeroed),
    so that many calls on a large n do not each allocate n bytes."""
    out = np.empty(tau, dtype=np.int32)
    if workspace is not None and (workspace.dtype != np.uint8 or workspace.size < n
                                  or not workspace.flags.c_contiguous):
        raise ValueError("workspace must be a contiguous zeroed uint8[n]")
    rc = _load().or_sample(seed, k, tau, n, _ptr(out), None if workspace is None else _ptr(workspace))
    if rc != 0:
        raise ValueError("or_sample failed (rc=%d)" % rc)
    return out


def samples(seed: int, k0: int, count: int, tau: int, n: int) -> np.ndarray:
    """O5 for k = k0 .. k0+count-1: int32[count, tau], row k-k0 = slot array of S_k."""
    ws = np.zeros(n, dtype=np.uint8)
    out = np.empty((count, tau), dtype=np.int32)
    for t in range(count):
        out[t] = sample(seed, k0 + t, tau, n, workspace=ws)
    return out


# ---------------------------------------------------------------- other DU samplings (NEXT-1)
KINDS = {"nice": 0, "independent": 1, "binomial": 2, "du": 3}


class Sampling:
    """A doubly uniform sampling: kind in KINDS, tau processors /
    slots, p_b for binomial, q[0..tau] (size law) for du."""

    def __init__(self, kind="nice", tau=1, p_b=1.0, q=None):
        self.kind, self.tau, self.p_b = kind, int(tau), float(p_b)
        self.q = None if q is None else np.ascontiguousarray(q, dtype=np.float64)
        if kind == "du" and (self.q is None or self.q.size != self.tau + 1):
            raise ValueError("du sampling needs q[0..tau]")

    def _q(self):
        return _ptr(self.q) if self.q is not None else None


def sample_kind(s: Sampling, seed: int, k: int, n: int) -> np.ndarray:
    """Slot array of S_k for sampling s (idle slots are -1)."""
    out = np.empty(s.tau, dtype=np.int32)
    rc = _load().or_sample_kind(KINDS[s.kind], seed, k, s.tau, n, s.p_b, s._q(), _ptr(out))
    if rc != 0:
        raise ValueError("or_sample_kind failed (rc=%d)" % rc)
    return out


def moments(s: Sampling, n: int):
    """(E|S|, E|S|^2) of the sampling."""
    e1, e2 = ctypes.c_double(), ctypes.c_double()
    rc = _load().or_moments(KINDS[s.kind], s.tau, n, s.p_b, s._q(), ctypes.byref(e1), ctypes.byref(e2))
    if rc != 0:
        raise ValueError("or_moments failed")
    return e1.value, e2.value


def beta_du(omega_: int, n: int, e1: float, e2: float) -> float:
    """thm:ESO-DU: beta = 1 + (omega-1)(E|S|^2/E|S| - 1)/max(1,n-1)."""
    return float(_load().or_beta_du(omega_, n, e1, e2))


def beta_sampling(omega_: int, n: int, s: Sampling) -> float:
    return beta_du(omega_, n, *moments(s, n))


def row_counts(m: int, rowidx) -> np.ndarray:
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    counts = np.zeros(m, dtype=np.int64)
    _load().or_row_counts(rowidx.size, _ptr(rowidx), _ptr(counts))
    return counts


def omega(m: int, rowidx) -> int:
    """O1: max stored entries in any row."""
    rowidx = np.ascontiguousarray(rowidx, dtype=np.int32)
    return int(_load().or_omega(m, rowidx.size, _ptr(rowidx)))


def col_norms(colptr, val) -> np.ndarray:
    """O2: L_i = ||a_i||^2 in fp64."""
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float32)
    n = colptr.size - 1
    L = np.empty(n, dtype=np.float64)
    _load().or_col_norms(n, _ptr(colptr), _ptr(val), _ptr(L))
    return L


def beta(omega_: int, tau: int, n: int) -> float:
    """O3: beta = 1 + (omega-1)(tau-1)/max(1,n-1)."""
    return float(_load().or_beta(omega_, tau, n))


def prox(x: float, g: float, s: float, lam: float) -> float:
    """Soft-threshold block update: returns x+ = x + h_i."""
    return float(_load().or_prox(x, g, s, lam))


def residual(m, colptr, rowidx, val, b, x) -> np.ndarray:
    """O4: r = Ax - b in fp64."""
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    b = np.ascontiguousarray(b, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    r = np.empty(m, dtype=np.float64)
    _load().or_residual(m, colptr.size - 1, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(b),
                        _ptr(x), _ptr(r))
    return r


def objective(m, colptr, rowidx, val, b, lam, x) -> float:
    """F(x) = 1/2||Ax-b||^2 + lambda||x||_1 in fp64."""
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    b = np.ascontiguousarray(b, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_load().or_objective(m, colptr.size - 1, _ptr(colptr), _ptr(rowidx), _ptr(val),
                                      _ptr(b), lam, _ptr(x)))


def refresh_period(n: int, tau: int, refresh_every: int = 0) -> int:
    return int(_load().or_refresh_period(n, tau, refresh_every))


class RunResult:
    __slots__ = ("x", "r", "slots", "loop_seconds", "omega", "beta", "L")

    def __init__(self, x, r, slots, loop_seconds, omega_, beta_, L):
        self.x, self.r, self.slots, self.loop_seconds = x, r, slots, loop_seconds
        self.omega, self.beta, self.L = omega_, beta_, L


def run(m, colptr, rowidx, val, b, lam, tau, iters, seed, x0=None, first_iter=0,
        refresh_every=0, beta_override=None, omega_override=None, L=None,
        keep_slots=False, sampling: Sampling = None) -> RunResult:
    """Synchronous PCDM1 (alg:PCD1) for LASSO, O1..O8 of SURVEY 8(c).

    omega_override / L let a caller hand in the oracle's own omega / L computed
    on a larger matrix (sub-instance runs); they never come from the GPU path.
    """
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    b = np.ascontiguousarray(b, dtype=np.float32)
    n = colptr.size - 1
    lib = _load()
    om = omega(m, rowidx) if omega_override is None else int(omega_override)
    Lv = col_norms(colptr, val) if L is None else np.ascontiguousarray(L, dtype=np.float64)
    if sampling is not None:
        tau = sampling.tau
    if beta_override is not None:
        bt = float(beta_override)
    elif sampling is None or sampling.kind == "nice":
        bt = beta(om, tau, n)
    else:
        bt = beta_sampling(om, n, sampling)
    x = np.zeros(n, dtype=np.float64) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    r = np.empty(m, dtype=np.float64)
    slots = np.empty(iters * tau, dtype=np.int32) if keep_slots else None
    secs = ctypes.c_double(0.0)
    if sampling is None or sampling.kind == "nice":
        rc = lib.or_run(m, n, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(b), lam, _ptr(Lv), bt,
                        _ptr(x), tau, iters, seed, first_iter, refresh_every, _ptr(r),
                        _ptr(slots) if keep_slots else None, ctypes.byref(secs))
    else:
        rc = lib.or_run_kind(m, n, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(b), lam, _ptr(Lv), bt,
                             _ptr(x), KINDS[sampling.kind], tau, sampling.p_b, sampling._q(), iters, seed,
                             first_iter, refresh_every, _ptr(r), _ptr(slots) if keep_slots else None,
                             ctypes.byref(secs))
    if rc < 0:
        raise ValueError("or_run failed (rc=%d)" % rc)
    if rc == 1:
        raise FloatingPointError("oracle: non-finite delta (diverged)")
    return RunResult(x, r, slots.reshape(iters, tau) if keep_slots else None, secs.value, om, bt, Lv)


# ---------------------------------------------------------------- L2-regularised logistic regression (NEXT-3)
def margins(m, colptr, rowidx, val, y, x) -> np.ndarray:
    """s_j = y_j (Ax)_j in fp64."""
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    y = np.ascontiguousarray(y, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    s = np.empty(m, dtype=np.float64)
    _load().or_margins(m, colptr.size - 1, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(y), _ptr(x), _ptr(s))
    return s


def logistic_objective(m, colptr, rowidx, val, y, lam, x) -> float:
    """F(x) = sum_j log(1 + exp(-y_j A_j^T x)) + lambda ||x||^2 (Sec. 8.4)."""
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    y = np.ascontiguousarray(y, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_load().or_logistic_objective(m, colptr.size - 1, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(y),
                                               lam, _ptr(x)))


def logistic_grad_i(colptr, rowidx, val, y, s, i) -> float:
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    y = np.ascontiguousarray(y, dtype=np.float32)
    s = np.ascontiguousarray(s, dtype=np.float64)
    return float(_load().or_logistic_grad_i(_ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(y), _ptr(s), i))


def logistic_L(colptr, val) -> np.ndarray:
    colptr = np.ascontiguousarray(colptr, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float32)
    n = colptr.size - 1
    L = np.empty(n, dtype=np.float64)
    _load().or_logistic_L(n, _ptr(colptr), _ptr(val), _ptr(L))
    return L


def logistic_step(x, g, s, lam) -> float:
    return float(_load().or_logistic_step(x, g, s, lam))


def logistic_run(m, colptr, rowidx, val, y, lam, tau, iters, seed, x0=None, first_iter=0, refresh_every=0,
                 beta_override=None, sampling: Sampling = None):
    """Synchronous PCDM1 on the L2-regularised logistic problem (O5-O8 with margins)."""
    colptr, rowidx, val = _csc(colptr, rowidx, val)
    y = np.ascontiguousarray(y, dtype=np.float32)
    n = colptr.size - 1
    om = omega(m, rowidx)
    L = logistic_L(colptr, val)
    S = sampling if sampling is not None else Sampling("nice", tau)
    bt = float(beta_override) if beta_override is not None else (
        beta(om, S.tau, n) if S.kind == "nice" else beta_sampling(om, n, S))
    x = np.zeros(n, dtype=np.float64) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    s = np.empty(m, dtype=np.float64)
    secs = ctypes.c_double(0.0)
    rc = _load().or_logistic_run(m, n, _ptr(colptr), _ptr(rowidx), _ptr(val), _ptr(y), lam, _ptr(L), bt, _ptr(x),
                                 KINDS[S.kind], S.tau, S.p_b, S._q(), iters, seed, first_iter, refresh_every,
                                 _ptr(s), ctypes.byref(secs))
    if rc < 0:
        raise ValueError("or_logistic_run failed (rc=%d)" % rc)
    if rc == 1:
        raise FloatingPointError("oracle: non-finite step")
    return RunResult(x, s, None, secs.value, om, bt, L)
