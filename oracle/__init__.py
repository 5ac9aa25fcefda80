"""ctypes binding for the fp64 CPU oracle (oracle/nndtw_oracle.c).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The CUDA product path
(paper_1808_09617_b200) never imports it and shares no code with it.

Every function takes numpy arrays; float inputs are converted to contiguous float32 (the
product's storage type) and promoted to double inside the C code.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nndtw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread",
          "-std=c11", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (building the checker is not using it)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


class Counts(C.Structure):
    _fields_ = [("lb_calls", C.c_int64), ("pruned_kim", C.c_int64),
                ("pruned_enh", C.c_int64), ("dtw_calls", C.c_int64),
                ("dtw_abandoned", C.c_int64), ("cells", C.c_int64)]


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = C.CDLL(build())
        fp = C.POINTER(C.c_float)
        dp = C.POINTER(C.c_double)
        i64p = C.POINTER(C.c_int64)
        i32p = C.POINTER(C.c_int32)
        ip = C.POINTER(C.c_int)
        lib.oracle_dtw.restype = C.c_double
        lib.oracle_dtw.argtypes = [fp, fp, C.c_int, C.c_int]
        lib.oracle_dtw_cut.restype = C.c_double
        lib.oracle_dtw_cut.argtypes = [fp, fp, C.c_int, C.c_int, C.c_double, ip, i64p]
        lib.oracle_sqed.restype = C.c_double
        lib.oracle_sqed.argtypes = [fp, fp, C.c_int]
        lib.oracle_envelope.restype = None
        lib.oracle_envelope.argtypes = [fp, C.c_int, C.c_int, fp, fp]
        lib.oracle_envelopes.restype = None
        lib.oracle_envelopes.argtypes = [fp, C.c_int64, C.c_int, C.c_int, fp, fp]
        lib.oracle_lb_kim_sum.restype = C.c_double
        lib.oracle_lb_kim_sum.argtypes = [fp, fp, C.c_int]
        lib.oracle_lb_keogh.restype = C.c_double
        lib.oracle_lb_keogh.argtypes = [fp, fp, fp, C.c_int]
        lib.oracle_lb_enhanced.restype = C.c_double
        lib.oracle_lb_enhanced.argtypes = [fp, fp, fp, fp, C.c_int, C.c_int, C.c_int,
                                           C.c_double, C.c_double, ip]
        lib.oracle_lb_cascade.restype = C.c_double
        lib.oracle_lb_cascade.argtypes = [fp, fp, fp, fp, C.c_int, C.c_int, C.c_int]
        lib.oracle_lb_improved.restype = C.c_double
        lib.oracle_lb_improved.argtypes = [fp, fp, fp, fp, C.c_int, C.c_int]
        lib.oracle_lb_new.restype = C.c_double
        lib.oracle_lb_new.argtypes = [fp, fp, C.c_int, C.c_int]
        lib.oracle_lb_enhanced_improved.restype = C.c_double
        lib.oracle_lb_enhanced_improved.argtypes = [fp, fp, fp, fp, C.c_int, C.c_int, C.c_int]
        lib.oracle_lb_enhanced_sym.restype = C.c_double
        lib.oracle_lb_enhanced_sym.argtypes = [fp, fp, fp, fp, fp, fp, C.c_int, C.c_int,
                                               C.c_int]
        lib.oracle_nn.restype = None
        lib.oracle_nn.argtypes = [fp, C.c_int64, fp, fp, fp, C.c_int64, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, i64p, dp, C.POINTER(Counts)]
        lib.oracle_loocv.restype = None
        lib.oracle_loocv.argtypes = [fp, i32p, C.c_int64, C.c_int, i32p, C.c_int, C.c_int,
                                     C.c_int64, C.c_int64, C.c_int, C.c_int, i64p, i64p]
        _lib = lib
        return lib


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def dtw(a, b, w: int, cutoff: float = float("inf")) -> float:
    """Squared DTW_W (Eq. 1); +inf if abandoned at `cutoff` (row-min test)."""
    a, b = _f32(a), _f32(b)
    assert a.shape == b.shape and a.ndim == 1
    lib = _load()
    ab = C.c_int(0)
    return lib.oracle_dtw_cut(_ptr(a, C.c_float), _ptr(b, C.c_float), a.size, int(w),
                              float(cutoff), C.byref(ab), None)


def dtw_cut(a, b, w: int, cutoff: float):
    a, b = _f32(a), _f32(b)
    lib = _load()
    ab = C.c_int(0)
    cells = C.c_int64(0)
    d = lib.oracle_dtw_cut(_ptr(a, C.c_float), _ptr(b, C.c_float), a.size, int(w),
                           float(cutoff), C.byref(ab), C.byref(cells))
    return d, bool(ab.value), int(cells.value)


def sqed(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return _load().oracle_sqed(_ptr(a, C.c_float), _ptr(b, C.c_float), a.size)


def envelope(b, w: int):
    b = _f32(b)
    U = np.empty_like(b)
    Lo = np.empty_like(b)
    _load().oracle_envelope(_ptr(b, C.c_float), b.size, int(w), _ptr(U, C.c_float),
                            _ptr(Lo, C.c_float))
    return U, Lo


def envelopes(X, w: int):
    X = _f32(X)
    n, L = X.shape
    U = np.empty_like(X)
    Lo = np.empty_like(X)
    _load().oracle_envelopes(_ptr(X, C.c_float), n, L, int(w), _ptr(U, C.c_float),
                             _ptr(Lo, C.c_float))
    return U, Lo


def lb_kim_sum(a, b) -> float:
    a, b = _f32(a), _f32(b)
    return _load().oracle_lb_kim_sum(_ptr(a, C.c_float), _ptr(b, C.c_float), a.size)


def lb_keogh(a, U, Lo) -> float:
    a, U, Lo = _f32(a), _f32(U), _f32(Lo)
    return _load().oracle_lb_keogh(_ptr(a, C.c_float), _ptr(U, C.c_float),
                                   _ptr(Lo, C.c_float), a.size)


def lb_enhanced(a, b, U, Lo, w: int, V: int, D: float = float("inf"), margin: float = 0.0):
    """Algorithm 1.  Returns (value, aborted)."""
    a, b, U, Lo = _f32(a), _f32(b), _f32(U), _f32(Lo)
    ab = C.c_int(0)
    v = _load().oracle_lb_enhanced(_ptr(a, C.c_float), _ptr(b, C.c_float), _ptr(U, C.c_float),
                                   _ptr(Lo, C.c_float), a.size, int(w), int(V), float(D),
                                   float(margin), C.byref(ab))
    return v, bool(ab.value)


def lb_cascade(a, b, U, Lo, w: int, V: int) -> float:
    a, b, U, Lo = _f32(a), _f32(b), _f32(U), _f32(Lo)
    return _load().oracle_lb_cascade(_ptr(a, C.c_float), _ptr(b, C.c_float),
                                     _ptr(U, C.c_float), _ptr(Lo, C.c_float), a.size, int(w),
                                     int(V))


def lb_improved(a, b, w: int, UB=None, LB=None) -> float:
    """LB_Improved_W(A, B); envelope of B computed here unless given."""
    a, b = _f32(a), _f32(b)
    if UB is None:
        UB, LB = envelope(b, w)
    UB, LB = _f32(UB), _f32(LB)
    return _load().oracle_lb_improved(_ptr(a, C.c_float), _ptr(b, C.c_float),
                                      _ptr(UB, C.c_float), _ptr(LB, C.c_float), a.size, int(w))


def lb_new(a, b, w: int) -> float:
    """LB_New_W(A, B)."""
    a, b = _f32(a), _f32(b)
    return _load().oracle_lb_new(_ptr(a, C.c_float), _ptr(b, C.c_float), a.size, int(w))


def lb_enhanced_improved(a, b, w: int, V: int, UB=None, LB=None) -> float:
    """LB_Enhanced^V with the LB_Improved bridge (reading C21)."""
    a, b = _f32(a), _f32(b)
    if UB is None:
        UB, LB = envelope(b, w)
    UB, LB = _f32(UB), _f32(LB)
    return _load().oracle_lb_enhanced_improved(_ptr(a, C.c_float), _ptr(b, C.c_float),
                                               _ptr(UB, C.c_float), _ptr(LB, C.c_float),
                                               a.size, int(w), int(V))


def lb_enhanced_sym(a, b, w: int, V: int) -> float:
    """max(LB_Enhanced(A,B), LB_Enhanced(B,A))."""
    a, b = _f32(a), _f32(b)
    UA, LA = envelope(a, w)
    UB, LB = envelope(b, w)
    return _load().oracle_lb_enhanced_sym(_ptr(a, C.c_float), _ptr(b, C.c_float),
                                          _ptr(UA, C.c_float), _ptr(LA, C.c_float),
                                          _ptr(UB, C.c_float), _ptr(LB, C.c_float), a.size,
                                          int(w), int(V))


def bound_matrix(kind: str, Q, T, w: int, V: int = 5) -> np.ndarray:
    """All-pairs bound matrix [nq][nt] (fp64) for kind in {keogh, enhanced, cascade, sym,
    improved, new, enhanced_improved}; plain loops over the single-pair functions above (small inputs only)."""
    Q, T = _f32(Q), _f32(T)
    UT, LT = envelopes(T, w)
    out = np.empty((Q.shape[0], T.shape[0]), dtype=np.float64)
    for i, a in enumerate(Q):
        for j, b in enumerate(T):
            if kind == "keogh":
                out[i, j] = lb_keogh(a, UT[j], LT[j])
            elif kind == "enhanced":
                out[i, j] = lb_enhanced(a, b, UT[j], LT[j], w, V)[0]
            elif kind == "cascade":
                out[i, j] = lb_cascade(a, b, UT[j], LT[j], w, V)
            elif kind == "sym":
                out[i, j] = lb_enhanced_sym(a, b, w, V)
            elif kind == "improved":
                out[i, j] = lb_improved(a, b, w, UT[j], LT[j])
            elif kind == "new":
                out[i, j] = lb_new(a, b, w)
            elif kind == "enhanced_improved":
                out[i, j] = lb_enhanced_improved(a, b, w, V, UT[j], LT[j])
            else:
                raise ValueError(kind)
    return out


def tightness(lb, dtw) -> tuple[float, int]:
    """Mean tightness sqrt(LB)/sqrt(DTW^2) over pairs with DTW > 0 (reading C20)."""
    lb = np.asarray(lb, dtype=np.float64).ravel()
    d = np.asarray(dtw, dtype=np.float64).ravel()
    m = d > 0
    return float(np.mean(np.sqrt(lb[m]) / np.sqrt(d[m]))) if m.any() else 0.0, int(m.sum())


def nn(Q, T, w: int, V: int = 5, mode: str = "exhaustive", threads: int | None = None,
       envelopes_UL=None, with_counts: bool = False):
    """1-NN of every query.  mode 'exhaustive' (i) or 'pruned' (ii, the paper's search)."""
    Q, T = _f32(Q), _f32(T)
    nq, L = Q.shape
    nt = T.shape[0]
    m = 0 if mode == "exhaustive" else 1
    if m == 1:
        if envelopes_UL is None:
            U, Lo = envelopes(T, w)
        else:
            U, Lo = (_f32(e) for e in envelopes_UL)
    else:
        U = Lo = T  # not read
    idx = np.empty(nq, dtype=np.int64)
    dist = np.empty(nq, dtype=np.float64)
    counts = (Counts * max(nq, 1))()
    _load().oracle_nn(_ptr(Q, C.c_float), nq, _ptr(T, C.c_float), _ptr(U, C.c_float),
                      _ptr(Lo, C.c_float), nt, L, int(w), int(V), m,
                      threads or default_threads(), _ptr(idx, C.c_int64),
                      _ptr(dist, C.c_double), counts)
    if with_counts:
        cnt = {f: np.array([getattr(counts[i], f) for i in range(nq)], dtype=np.int64)
               for f, _ in Counts._fields_}
        return idx, dist, cnt
    return idx, dist


def loocv(X, labels, windows, V: int = 5, q_begin: int = 0, q_end: int | None = None,
          mode: str = "pruned", threads: int | None = None):
    """Leave-one-out error counts per window; returns (errors[nw], nn[nw][nq])."""
    X = _f32(X)
    labels = np.ascontiguousarray(np.asarray(labels, dtype=np.int32))
    n, L = X.shape
    q_end = n if q_end is None else q_end
    win = np.ascontiguousarray(np.asarray(windows, dtype=np.int32))
    nw = win.size
    errors = np.zeros(nw, dtype=np.int64)
    nn_out = np.empty((nw, max(q_end - q_begin, 0)), dtype=np.int64)
    _load().oracle_loocv(_ptr(X, C.c_float), _ptr(labels, C.c_int32), n, L,
                         _ptr(win, C.c_int32), nw, int(V), q_begin, q_end,
                         0 if mode == "exhaustive" else 1, threads or default_threads(),
                         _ptr(errors, C.c_int64), _ptr(nn_out, C.c_int64))
    return errors, nn_out
