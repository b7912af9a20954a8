"""CPU oracle for the PLSSVM hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this package.  The product package ``paper_2202_12674_b200``
never imports it, and it never imports the product package.

The arithmetic lives in ``oracle.c`` (plain C, fp64, sequential sums, OpenMP only over
independent rows); this module only loads it and marshals numpy arrays.  Each function
cites the passage it follows (P:L = PAPER.md line L, S:L = SPEC.md line L).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_lib = None


def _host_tag() -> str:
    """-march=native code is specific to the host CPU: one build per CPU model / flag set (the repo
    snapshot travels to the GPU box, whose host may not run this machine's instructions)."""
    import hashlib

    key = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith(("model name", "flags")):
                    key += ln
                if ln.startswith("flags"):
                    break
    except OSError:
        pass
    return hashlib.sha1(key.encode()).hexdigest()[:10]


_LIB = os.path.join(_HERE, f"liboracle_{_host_tag()}.so")

LINEAR, POLYNOMIAL, RBF = 0, 1, 2
OK, E_INVALID, E_NUMERICAL, W_NOT_CONVERGED = 0, 1, 6, 7


def build(force: bool = False) -> str:
    """Compile oracle.c: -O3 -march=native (SURVEY §8(d) oracle-timing protocol), ISO C11 with
    -ffp-contract=off and no fast-math (every rounding is the one the source spells out), OpenMP
    over independent rows only."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = f"{_LIB}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ct.CDLL(_LIB)
        dp, i64, i32p = ct.POINTER(ct.c_double), ct.c_int64, ct.POINTER(ct.c_int32)
        lib.oracle_kernel.restype = ct.c_double
        lib.oracle_kernel.argtypes = [dp, dp, i64, ct.c_int, ct.c_double, ct.c_int, ct.c_double]
        lib.oracle_q.argtypes = [dp, i64, i64, ct.c_int, ct.c_double, ct.c_int, ct.c_double, ct.c_double, dp, dp]
        lib.oracle_qtilde.argtypes = [dp, i64, i64, ct.c_int, ct.c_double, ct.c_int, ct.c_double, ct.c_double, dp]
        lib.oracle_qtilde_rows.argtypes = [dp, i64, i64, ct.c_int, ct.c_double, ct.c_int, ct.c_double,
                                           ct.c_double, ct.POINTER(ct.c_int64), i64, dp]
        lib.oracle_matvec.argtypes = [dp, i64, dp, dp]
        lib.oracle_cg.restype = ct.c_int
        lib.oracle_cg.argtypes = [dp, i64, dp, dp, ct.c_double, i64, i64, ct.POINTER(ct.c_int64), dp]
        lib.oracle_train.restype = ct.c_int
        lib.oracle_train.argtypes = [dp, dp, i64, i64, ct.c_int, ct.c_double, ct.c_int, ct.c_double,
                                     ct.c_double, ct.c_double, i64, ct.c_int, i64, dp, dp,
                                     ct.POINTER(ct.c_int64), dp]
        lib.oracle_predict.argtypes = [dp, dp, ct.c_double, i64, i64, ct.c_int, ct.c_double, ct.c_int,
                                       ct.c_double, dp, i64, dp, i32p]
        lib.oracle_num_threads.restype = ct.c_int
        _lib = lib
    return _lib


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return a.ctypes.data_as(ct.POINTER(ct.c_double))


def num_threads() -> int:
    return _load().oracle_num_threads()


def kernel(a, b, kernel_id, gamma=1.0, degree=3, coef0=0.0) -> float:
    """k(a, b)."""
    a, b = _f64(a), _f64(b)
    return _load().oracle_kernel(_p(a), _p(b), a.size, kernel_id, gamma, degree, coef0)


def q_cache(X, kernel_id, gamma=1.0, degree=3, coef0=0.0, C=1.0):
    """(q, Q_mm), P:391-395 and Eq. 12 (x_m = last point)."""
    X = _f64(X)
    m, d = X.shape
    q = np.empty(m - 1)
    Qmm = ct.c_double()
    _load().oracle_q(_p(X), m, d, kernel_id, gamma, degree, coef0, C, _p(q), ct.byref(Qmm))
    return q, Qmm.value


def qtilde(X, kernel_id, gamma=1.0, degree=3, coef0=0.0, C=1.0):
    """Explicit Q~ (m-1)x(m-1), Eq. 13/16."""
    X = _f64(X)
    m, d = X.shape
    Qt = np.empty((m - 1, m - 1))
    _load().oracle_qtilde(_p(X), m, d, kernel_id, gamma, degree, coef0, C, _p(Qt))
    return Qt


def qtilde_rows(X, rows, kernel_id, gamma=1.0, degree=3, coef0=0.0, C=1.0):
    """Rows of Q~ (Eq. 16) without forming the whole matrix."""
    X = _f64(X)
    m, d = X.shape
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.empty((rows.size, m - 1))
    _load().oracle_qtilde_rows(_p(X), m, d, kernel_id, gamma, degree, coef0, C,
                               rows.ctypes.data_as(ct.POINTER(ct.c_int64)), rows.size, _p(out))
    return out


def matvec(A, p):
    """y = A p (plain row sums)."""
    A, p = _f64(A), _f64(p)
    n = p.size
    y = np.empty(n)
    _load().oracle_matvec(_p(A), n, _p(p), _p(y))
    return y


def cg(A, b, eps=1e-10, imax=None, x0=None, replace_every=0, trace=False):
    """Shewchuk B2 CG (R-5).  Returns (x, iterations, status[, trace])."""
    A, b = _f64(A), _f64(b)
    n = b.size
    x = np.zeros(n) if x0 is None else _f64(x0).copy()
    imax = n if imax is None else imax
    it = ct.c_int64()
    tr = np.zeros(imax + 1) if trace else None
    st = _load().oracle_cg(_p(A), n, _p(b), _p(x), eps, imax, replace_every, ct.byref(it),
                           _p(tr) if trace else None)
    if trace:
        return x, it.value, st, tr[: it.value + 1]
    return x, it.value, st


def train(X, y, kernel_id, gamma=1.0, degree=3, coef0=0.0, C=1.0, eps=1e-10, imax=0, x0=0,
          replace_every=0, timings=False):
    """LS-SVM training via Eq. 12-16 + CG.  Returns (alpha[m], b, iterations, status[, timings])."""
    X, y = _f64(X), _f64(y)
    m, d = X.shape
    alpha = np.empty(m)
    b = ct.c_double()
    it = ct.c_int64()
    tm = np.zeros(3)
    st = _load().oracle_train(_p(X), _p(y), m, d, kernel_id, gamma, degree, coef0, C, eps, imax, x0,
                              replace_every, _p(alpha), ct.byref(b), ct.byref(it), _p(tm))
    if timings:
        return alpha, b.value, it.value, st, tm
    return alpha, b.value, it.value, st


def predict(X, alpha, b, Z, kernel_id, gamma=1.0, degree=3, coef0=0.0):
    """f(z) = sum alpha_i k(x_i, z) + b and labels (f >= 0 -> +1), Eq. 10."""
    X, alpha, Z = _f64(X), _f64(alpha), _f64(Z)
    m, d = X.shape
    n = Z.shape[0]
    f = np.empty(n)
    lab = np.empty(n, dtype=np.int32)
    _load().oracle_predict(_p(X), _p(alpha), b, m, d, kernel_id, gamma, degree, coef0, _p(Z), n, _p(f),
                           lab.ctypes.data_as(ct.POINTER(ct.c_int32)))
    return f, lab


def matvec_implicit(X, p, kernel_id, gamma=1.0, degree=3, coef0=0.0, C=1.0):
    """Q~ p with Q~ formed explicitly (small m only)."""
    return matvec(qtilde(X, kernel_id, gamma, degree, coef0, C), p)
