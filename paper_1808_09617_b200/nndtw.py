"""Thin Python binding of libnndtw.so (include/nndtw.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; PyTorch provides device memory,
streams and (in dist.py) process groups.  There is no CPU fallback: if the shared library is
missing or the device is not sm_100, the calls raise.

Names follow the C ABI: envelopes, series_stats, lb_enhanced, dtw_batch, classify,
classify_refine, classify_resolve, finalize, loocv_window.  Distances are squared (Eq. 1-2).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NNDTW_LIB") or os.path.join(
    _HERE, "libnndtw_debug.so" if os.environ.get("NNDTW_DEBUG") == "1" else "libnndtw.so")

NNDTW_LB_WITH_KIM = 1
NNDTW_LB_PARTIAL = 4
NNDTW_LB_KEOGH = 2
NNDTW_CLASSIFY_EXACT = 1
NNDTW_CLASSIFY_BOUND_KEOGH = 2
NNDTW_CLASSIFY_BOUND_SYMMETRIC = 4
NNDTW_CLASSIFY_PHASE_SEED = 8
NNDTW_CLASSIFY_PHASE_SEARCH = 16
NNDTW_CLASSIFY_PHASE_SEARCH_A = 32
NNDTW_CLASSIFY_PHASE_SEARCH_B = 64
NNDTW_CLASSIFY_LEVEL_STATS = 128
NNDTW_CLASSIFY_BOUND_IMPROVED = 256
NNDTW_CLASSIFY_BOUND_NEW = 512
NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED = 1024
NNDTW_CLASSIFY_BOUND_NONE = 2048
# S2 bound of Model(bound=...) -> classify flag
BOUND_FLAGS = {"enhanced": 0, "keogh": NNDTW_CLASSIFY_BOUND_KEOGH,
               "improved": NNDTW_CLASSIFY_BOUND_IMPROVED, "new": NNDTW_CLASSIFY_BOUND_NEW,
               "enhanced_improved": NNDTW_CLASSIFY_BOUND_ENHANCED_IMPROVED,
               "none": NNDTW_CLASSIFY_BOUND_NONE}
KEY_INIT = 0x7F800000FFFFFFFF


class NNDTWError(RuntimeError):
    pass


class Stats(C.Structure):
    _fields_ = [("lb_pairs", C.c_int64), ("survivors", C.c_int64), ("pruned_kim", C.c_int64),
                ("pruned_bands", C.c_int64), ("pruned_keogh", C.c_int64),
                ("bridge_pairs", C.c_int64), ("dtw_calls", C.c_int64),
                ("dtw_abandoned", C.c_int64), ("cells", C.c_int64),
                ("near_tie_pairs", C.c_int64), ("rounds", C.c_int32), ("launches", C.c_int32),
                ("ms_envelopes", C.c_float), ("ms_lb", C.c_float), ("ms_dtw", C.c_float),
                ("ms_other", C.c_float), ("ms_lb_bridge", C.c_float),
                ("dtw_fallback", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


def merge_stat_dicts(a: dict, b: dict) -> dict:
    """Sum two stats dicts; the per-level prune counters stay -1 (not computed) unless one
    side has them."""
    out = {}
    for k in a:
        if k.startswith("pruned_"):
            out[k] = -1 if a[k] < 0 and b[k] < 0 else max(a[k], 0) + max(b[k], 0)
        else:
            out[k] = a[k] + b[k]
    return out


_lib = None
_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32

_SIGS = {
    "nndtw_last_error": (C.c_char_p, []),
    "nndtw_version": (C.c_int, []),
    "nndtw_launch_count": (_I64, []),
    "nndtw_check_device": (C.c_int, []),
    "nndtw_dtw_kernel_name": (C.c_char_p, [_I32, _I32]),
    "nndtw_band_limited_window": (_I32, [_I32, _I32]),
    "nndtw_check_finite": (C.c_int, [_P, _I64, _P, _P]),
    "nndtw_envelopes": (C.c_int, [_P, _I64, _I32, _I32, _P, _P, _P, _P]),
    "nndtw_series_stats": (C.c_int, [_P, _I64, _I32, _P, _P]),
    "nndtw_lb_enhanced": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32,
                                    C.c_uint32, _P, _I64, _P]),
    "nndtw_lb_enhanced_symmetric": (C.c_int, [_P, _P, _P, _P, _I64, _P, _P, _P, _P, _I64, _I32,
                                              _I32, _I32, C.c_uint32, _P, _I64, _P]),
    "nndtw_lb_improved": (C.c_int, [_P, _I64, _P, _P, _P, _I64, _I32, _I32, _P, _I64, _P]),
    "nndtw_lb_enhanced_improved": (C.c_int, [_P, _I64, _P, _P, _P, _I64, _I32, _I32, _I32, _P,
                                             _I64, _P]),
    "nndtw_lb_new": (C.c_int, [_P, _I64, _P, _I64, _I32, _I32, _P, _I64, _P]),
    "nndtw_ed_seed_workspace_bytes": (C.c_size_t, [_I64, _I64, _I32]),
    "nndtw_ed_seed": (C.c_int, [_P, _I64, _P, _I64, _I32, _P, C.c_size_t, _P, _P]),
    "nndtw_tightness": (C.c_int, [_P, _P, _I64, _P, _P, _P, _P]),
    "nndtw_dtw_batch": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P]),
    "nndtw_classify_workspace_bytes": (C.c_size_t, [_I64, _I64, _I32, _I32]),
    "nndtw_classify_workspace_bytes_capped": (C.c_size_t, [_I64, _I64, _I32, _I32, _I64]),
    "nndtw_classify_overflowed": (C.c_int, [_P, C.c_size_t, _I64, _I64, _I32,
                                            C.POINTER(C.c_int32), _P]),
    "nndtw_classify": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _I32,
                                 C.c_uint32, _P, C.c_size_t, _P, C.POINTER(Stats), _P]),
    "nndtw_classify_refine": (C.c_int, [_P, C.c_size_t, _P, _I64, _P, _I64, _I32, _I32, _P,
                                        _P, _P]),
    "nndtw_classify_resolve": (C.c_int, [_P, C.c_size_t, _P, _I64, _P, _I64, _I32, _I32, _I64,
                                         _P, _P, _P, _P]),
    "nndtw_finalize": (C.c_int, [_P, _I64, _I32, _P, _I64, _P, _P, _P, _P]),
    "nndtw_loocv_workspace_bytes": (C.c_size_t, [_I64, _I32, _I64, _I64]),
    "nndtw_loocv_window": (C.c_int, [_P, _P, _I64, _I32, _P, _I32, _I32, _I64, _I64, _P,
                                     C.c_size_t, _P, _P, C.POINTER(Stats), _P]),
}

EXPORTED = tuple(_SIGS)


def load(path: str = LIB_PATH):
    """Load libnndtw.so (raises if it is missing -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NNDTWError(f"{path} not built; run paper_1808_09617_b200/build.py")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        msg = load().nndtw_last_error().decode(errors="replace")
        raise NNDTWError(f"{what} failed with code {rc}: {msg}")


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _series(x: torch.Tensor, name: str) -> torch.Tensor:
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32
            and x.dim() == 2 and x.is_contiguous()):
        raise NNDTWError(f"{name} must be a contiguous float32 CUDA tensor [n][L]")
    return x


def check_finite(x: torch.Tensor, stream=None) -> bool:
    bad = torch.zeros(1, dtype=torch.int32, device=x.device)
    _check(load().nndtw_check_finite(_ptr(x), x.numel(), _ptr(bad), _stream(stream)),
           "nndtw_check_finite")
    return int(bad.item()) == 0


def envelopes(x: torch.Tensor, w: int, with_kim: bool = True, stream=None):
    """S1: (upper, lower, kim) with kim an int32 tensor [n][4] = (vmin, vmax, imin, imax) bits."""
    _series(x, "x")
    n, L = x.shape
    U = torch.empty_like(x)
    Lo = torch.empty_like(x)
    kim = torch.empty((n, 4), dtype=torch.int32, device=x.device) if with_kim else None
    _check(load().nndtw_envelopes(_ptr(x), n, L, int(w), _ptr(U), _ptr(Lo), _ptr(kim),
                                  _stream(stream)), "nndtw_envelopes")
    return U, Lo, kim


def series_stats(x: torch.Tensor, stream=None) -> torch.Tensor:
    _series(x, "x")
    n, L = x.shape
    kim = torch.empty((n, 4), dtype=torch.int32, device=x.device)
    _check(load().nndtw_series_stats(_ptr(x), n, L, _ptr(kim), _stream(stream)),
           "nndtw_series_stats")
    return kim


def lb_enhanced(q, t, U, Lo, w: int, v: int, with_kim: bool = False, qkim=None, tkim=None,
                keogh: bool = False, stream=None, partial: bool = False) -> torch.Tensor:
    """S2: cascade bound matrix [nq][nt] (Eq. 7 / Algorithm 1; max with LB_Kim if asked;
    partial: Algorithm 1 up to its line-12 test -- boundary terms and bands, no bridge)."""
    _series(q, "q"); _series(t, "t"); _series(U, "U"); _series(Lo, "Lo")
    nq, L = q.shape
    nt = t.shape[0]
    if with_kim:
        qkim = series_stats(q, stream) if qkim is None else qkim
        if tkim is None:
            raise NNDTWError("tkim (from envelopes) is required with with_kim=True")
    out = torch.empty((nq, nt), dtype=torch.float32, device=q.device)
    _check(load().nndtw_lb_enhanced(_ptr(q), nq, _ptr(qkim), _ptr(t), _ptr(U), _ptr(Lo),
                                    _ptr(tkim), nt, L, int(w), int(v),
                                    (NNDTW_LB_WITH_KIM if with_kim else 0) |
                                    (NNDTW_LB_KEOGH if keogh else 0) |
                                    (NNDTW_LB_PARTIAL if partial else 0), _ptr(out), nt,
                                    _stream(stream)), "nndtw_lb_enhanced")
    return out


def lb_enhanced_symmetric(q, t, w: int, v: int, with_kim: bool = False, keogh: bool = False,
                          q_env=None, t_env=None, stream=None) -> torch.Tensor:
    """S2 symmetric bound matrix [nq][nt]: max(LB(q,t), LB(t,q))."""
    _series(q, "q"); _series(t, "t")
    nq, L = q.shape
    nt = t.shape[0]
    qU, qL, qk = q_env if q_env is not None else envelopes(q, w, with_kim, stream)
    tU, tL, tk = t_env if t_env is not None else envelopes(t, w, with_kim, stream)
    out = torch.empty((nq, nt), dtype=torch.float32, device=q.device)
    _check(load().nndtw_lb_enhanced_symmetric(
        _ptr(q), _ptr(qU), _ptr(qL), _ptr(qk if with_kim else None), nq, _ptr(t), _ptr(tU),
        _ptr(tL), _ptr(tk if with_kim else None), nt, L, int(w), int(v),
        (NNDTW_LB_WITH_KIM if with_kim else 0) | (NNDTW_LB_KEOGH if keogh else 0), _ptr(out),
        nt, _stream(stream)), "nndtw_lb_enhanced_symmetric")
    return out


def lb_improved(q, t, w: int, t_env=None, stream=None) -> torch.Tensor:
    """LB_Improved_W for all pairs [nq][nt]."""
    _series(q, "q"); _series(t, "t")
    nq, L = q.shape
    nt = t.shape[0]
    tU, tL = (t_env[0], t_env[1]) if t_env is not None else envelopes(t, w, False, stream)[:2]
    out = torch.empty((nq, nt), dtype=torch.float32, device=q.device)
    _check(load().nndtw_lb_improved(_ptr(q), nq, _ptr(t), _ptr(tU), _ptr(tL), nt, L, int(w),
                                    _ptr(out), nt, _stream(stream)), "nndtw_lb_improved")
    return out


def lb_enhanced_improved(q, t, w: int, v: int, t_env=None, stream=None) -> torch.Tensor:
    """LB_Enhanced^V with the LB_Improved bridge for all pairs [nq][nt]."""
    _series(q, "q"); _series(t, "t")
    nq, L = q.shape
    nt = t.shape[0]
    tU, tL = (t_env[0], t_env[1]) if t_env is not None else envelopes(t, w, False, stream)[:2]
    out = torch.empty((nq, nt), dtype=torch.float32, device=q.device)
    _check(load().nndtw_lb_enhanced_improved(_ptr(q), nq, _ptr(t), _ptr(tU), _ptr(tL), nt, L,
                                             int(w), int(v), _ptr(out), nt, _stream(stream)),
           "nndtw_lb_enhanced_improved")
    return out


def lb_new(q, t, w: int, stream=None) -> torch.Tensor:
    """LB_New_W for all pairs [nq][nt]."""
    _series(q, "q"); _series(t, "t")
    nq, L = q.shape
    nt = t.shape[0]
    out = torch.empty((nq, nt), dtype=torch.float32, device=q.device)
    _check(load().nndtw_lb_new(_ptr(q), nq, _ptr(t), nt, L, int(w), _ptr(out), nt,
                               _stream(stream)), "nndtw_lb_new")
    return out


def ed_seed(q, t, stream=None):
    """Euclidean-nearest train index of every query (int64 [nq]) and its squared ED as computed
    on piecewise-aggregate approximations (means over f points, ceil(L/f) <= 128; bf16 inputs,
    fp32 accumulation on the tensor cores) -- the paper's candidate order; a seed, not a
    distance."""
    _series(q, "q"); _series(t, "t")
    nq, L = q.shape
    nt = t.shape[0]
    lib = load()
    ws = torch.empty(lib.nndtw_ed_seed_workspace_bytes(nq, nt, L), dtype=torch.uint8,
                     device=q.device)
    key = torch.full((nq,), -1, dtype=torch.int64, device=q.device)
    _check(lib.nndtw_ed_seed(_ptr(q), nq, _ptr(t), nt, L, _ptr(ws), ws.numel(), _ptr(key),
                             _stream(stream)), "nndtw_ed_seed")
    idx = key & 0xFFFFFFFF
    dist = (key >> 32).to(torch.int32).view(torch.float32)
    return idx, dist


def tightness(lb: torch.Tensor, d: torch.Tensor, stream=None):
    """(mean of sqrt(lb/d) over pairs with 0 < d < inf, pair count, max ratio) -- P:37."""
    lb = lb.reshape(-1).contiguous()
    d = d.reshape(-1).contiguous()
    if lb.numel() != d.numel():
        raise NNDTWError("lb and dtw must have the same number of pairs")
    s = torch.zeros(1, dtype=torch.float64, device=lb.device)
    c = torch.zeros(1, dtype=torch.int64, device=lb.device)
    m = torch.zeros(1, dtype=torch.int32, device=lb.device)
    _check(load().nndtw_tightness(_ptr(lb), _ptr(d), lb.numel(), _ptr(s), _ptr(c), _ptr(m),
                                  _stream(stream)), "nndtw_tightness")
    cnt = int(c.item())
    mx = float(m.view(torch.float32).item())
    return (float(s.item()) / cnt if cnt else 0.0), cnt, mx


def dtw_batch(a, b, w: int, ia=None, ib=None, cutoff=None, stream=None) -> torch.Tensor:
    """S4: squared DTW_w of pairs (a[ia[p]], b[ib[p]]); +inf where abandoned at cutoff[p]."""
    _series(a, "a"); _series(b, "b")
    L = a.shape[1]
    if ia is not None:
        ia = ia.to(torch.int32).contiguous()
    if ib is not None:
        ib = ib.to(torch.int32).contiguous()
    npairs = ia.numel() if ia is not None else (ib.numel() if ib is not None else a.shape[0])
    if cutoff is not None:
        cutoff = cutoff.to(torch.float32).contiguous()
    out = torch.empty(npairs, dtype=torch.float32, device=a.device)
    _check(load().nndtw_dtw_batch(_ptr(a), _ptr(b), _ptr(ia), _ptr(ib), npairs, L, int(w),
                                  _ptr(cutoff), _ptr(out), _stream(stream)), "nndtw_dtw_batch")
    return out


@dataclass
class Prediction:
    idx: torch.Tensor     # int64 [nq] global train index of the 1-NN
    label: torch.Tensor   # int32 [nq]
    dist: torch.Tensor    # float32 [nq] squared DTW (sqrt for Eq. 2's DTW)
    stats: dict | None
    key: torch.Tensor | None = None  # int64 [nq] the packed keys (nndtw.classify)


class Model:
    """A train set with its envelopes and Kim features precomputed "at training time"."""

    def __init__(self, train: torch.Tensor, labels: torch.Tensor, w: int, v: int = 5,
                 index_base: int = 0, check: bool = True, stream=None, bound: str = "enhanced",
                 symmetric: bool = False):
        _series(train, "train")
        if check and not check_finite(train, stream):
            raise NNDTWError("train set contains NaN or infinity")
        self.t = train
        self.labels = labels.to(device=train.device, dtype=torch.int32).contiguous()
        self.L = train.shape[1]
        self.w = min(int(w), self.L - 1)
        self.v = int(v)
        self.index_base = int(index_base)
        if bound not in BOUND_FLAGS:
            raise NNDTWError(f"bound must be one of {sorted(BOUND_FLAGS)}")
        if symmetric and bound not in ("enhanced", "keogh"):
            raise NNDTWError("symmetric applies to the 'enhanced' and 'keogh' bounds only")
        self.bound = bound
        self.symmetric = bool(symmetric)
        self.U, self.Lo, self.kim = envelopes(train, self.w, True, stream)
        self._ws = None

    def workspace(self, nq: int, max_pairs: int | None = None) -> torch.Tensor:
        """Classify workspace for nq queries: the full layout, or (max_pairs) room for at most
        that many survivors / listed pairs (nndtw_classify_workspace_bytes_capped)."""
        lib = load()
        if max_pairs is None:
            need = lib.nndtw_classify_workspace_bytes(nq, self.t.shape[0], self.L, self.w)
        else:
            need = lib.nndtw_classify_workspace_bytes_capped(nq, self.t.shape[0], self.L, self.w,
                                                             int(max_pairs))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.t.device)
        return self._ws


def classify_keys(model: Model, q: torch.Tensor, exact: bool = True, self_offset: int = -1,
                  stats: bool = False, stream=None, phase: str | None = None, key=None, ws=None,
                  level_stats: bool = False, max_pairs: int | None = None):
    """S2-S7 on one shard: returns (key int64 [nq], workspace, stats dict | None).

    phase None runs everything; "seed" stops after the S3 seed round (keys = seed keys);
    "search" continues from a "seed" call's workspace `ws` with `key` = the MIN over shards
    of the seed keys (updated in place and returned); "search_a" / "search_b" split "search"
    in two (the lowest-bound survivors first), with another MIN over shards of `key` between."""
    _series(q, "q")
    nq, L = q.shape
    if L != model.L:
        raise NNDTWError("query length differs from train length (unequal lengths are out of "
                         "scope, reading C15)")
    if phase in ("search", "search_a", "search_b"):
        if ws is None or key is None:
            raise NNDTWError(f"phase {phase!r} needs the seed call's ws and the combined key")
    else:
        ws = model.workspace(nq, max_pairs)
        key = torch.empty(nq, dtype=torch.int64, device=q.device)
    flags = ((NNDTW_CLASSIFY_EXACT if exact else 0) |
             BOUND_FLAGS[model.bound] |
             (NNDTW_CLASSIFY_BOUND_SYMMETRIC if model.symmetric else 0) |
             (NNDTW_CLASSIFY_LEVEL_STATS if (stats and level_stats) else 0) |
             {None: 0, "seed": NNDTW_CLASSIFY_PHASE_SEED,
              "search": NNDTW_CLASSIFY_PHASE_SEARCH,
              "search_a": NNDTW_CLASSIFY_PHASE_SEARCH_A,
              "search_b": NNDTW_CLASSIFY_PHASE_SEARCH_B}[phase])
    st = Stats()
    _check(load().nndtw_classify(_ptr(q), nq, _ptr(model.t), _ptr(model.U), _ptr(model.Lo),
                                 _ptr(model.kim), model.t.shape[0], model.index_base,
                                 int(self_offset), L, model.w, model.v, flags,
                                 _ptr(ws), ws.numel(),
                                 _ptr(key), C.byref(st) if stats else None, _stream(stream)),
           "nndtw_classify")
    return key, ws, (st.as_dict() if stats else None)


def classify_overflowed(model: Model, nq: int, ws: torch.Tensor, stream=None) -> bool:
    """Whether the last classify on ws stored fewer survivors / listed pairs than it had (a
    capped workspace): its keys are then not valid.  Synchronises the stream."""
    out = C.c_int32(0)
    _check(load().nndtw_classify_overflowed(_ptr(ws), ws.numel(), nq, model.t.shape[0], model.L,
                                            C.byref(out), _stream(stream)),
           "nndtw_classify_overflowed")
    return bool(out.value)


def merge_stats(a: dict | None, b: dict | None) -> dict | None:
    """Sum two stats dicts (the seed and search phases of one sharded call)."""
    if a is None or b is None:
        return a or b
    return merge_stat_dicts(a, b)


def classify_refine(model: Model, q, ws, gkey, stream=None) -> torch.Tensor:
    nq = q.shape[0]
    f64 = torch.empty(nq, dtype=torch.int64, device=q.device)
    _check(load().nndtw_classify_refine(_ptr(ws), ws.numel(), _ptr(q), nq, _ptr(model.t),
                                        model.t.shape[0], model.L, model.w, _ptr(gkey),
                                        _ptr(f64), _stream(stream)), "nndtw_classify_refine")
    return f64


def classify_resolve(model: Model, q, ws, gkey, gf64, stream=None) -> torch.Tensor:
    nq = q.shape[0]
    out = torch.empty(nq, dtype=torch.int64, device=q.device)
    _check(load().nndtw_classify_resolve(_ptr(ws), ws.numel(), _ptr(q), nq, _ptr(model.t),
                                         model.t.shape[0], model.L, model.w, model.index_base,
                                         _ptr(gkey), _ptr(gf64), _ptr(out), _stream(stream)),
           "nndtw_classify_resolve")
    return out


def finalize(key, labels, key_format: int = 0, stream=None):
    nq = key.numel()
    idx = torch.empty(nq, dtype=torch.int64, device=key.device)
    lab = torch.empty(nq, dtype=torch.int32, device=key.device)
    dist = torch.empty(nq, dtype=torch.float32, device=key.device)
    _check(load().nndtw_finalize(_ptr(key), nq, int(key_format), _ptr(labels),
                                 labels.numel() if labels is not None else 0, _ptr(idx),
                                 _ptr(lab), _ptr(dist), _stream(stream)), "nndtw_finalize")
    return idx, lab, dist


WORKSPACE_BUDGET = 48 << 30  # bytes of classify workspace per call before queries are blocked
SURVIVOR_CAP = 0.125  # nndtw.classify: survivors / listed pairs reserved, as a fraction of pairs
CAP_MIN_PAIRS = 1 << 24  # calls with fewer (query, train) pairs keep the full layout by default


def classify(model: Model, q: torch.Tensor, stats: bool = False, check: bool = True,
             stream=None, workspace_budget: int | None = None,
             level_stats: bool = False, survivor_cap: float | None = None) -> Prediction:
    """Exact 1-NN of every query (single GPU / single shard, fp64-exact tie resolution).

    The workspace holds the 4-byte bound matrix per (query, train) pair and room for
    survivor_cap (default SURVIVOR_CAP) of the pairs as survivors and as two-stage list entries
    (20 bytes each; config 2 uses 3.6 % and 5.7 %) -- by default for calls above CAP_MIN_PAIRS
    pairs; smaller ones keep the full layout.  A call that needs more is detected
    (nndtw_classify_overflowed, one stream synchronisation per call) and rerun with the full
    layout (every pair: 24 bytes per pair); survivor_cap >= 1 uses the full layout directly.
    When the workspace exceeds `workspace_budget` (default 48 GB of the B200's 180 GB) the
    queries are processed in blocks -- queries are independent, the answer is the same."""
    if check and not check_finite(q, stream):
        raise NNDTWError("queries contain NaN or infinity")
    budget = WORKSPACE_BUDGET if workspace_budget is None else int(workspace_budget)
    frac = SURVIVOR_CAP if survivor_cap is None else float(survivor_cap)
    nq = q.shape[0]
    nt = model.t.shape[0]
    # (by default only large calls are capped: below 2^24 pairs the full layout is <= 400 MB and
    # a capped call would add a host synchronisation for nothing)
    capped = frac < 1.0 and (survivor_cap is not None or nq * nt > CAP_MIN_PAIRS)
    lib = load()

    def max_pairs(b: int) -> int | None:
        return int(frac * b * nt) + 1 if capped else None

    def ws_bytes(b: int) -> int:
        if capped:
            return lib.nndtw_classify_workspace_bytes_capped(b, nt, model.L, model.w, max_pairs(b))
        return lib.nndtw_classify_workspace_bytes(b, nt, model.L, model.w)

    blk = nq
    while blk > 1 and ws_bytes(blk) > budget:
        blk = (blk + 1) // 2
    keys, st = [], None
    for i in range(0, max(nq, 1), max(blk, 1)):
        qb = q[i:i + blk]
        k, ws, s = classify_keys(model, qb, exact=True, stats=stats, stream=stream,
                                 level_stats=level_stats, max_pairs=max_pairs(qb.shape[0]))
        if capped and qb.shape[0] > 0 and classify_overflowed(model, qb.shape[0], ws, stream):
            # more survivors than reserved: rerun this block with room for every pair
            pred = classify(model, qb, stats=stats, check=False, stream=stream,
                            workspace_budget=budget, level_stats=level_stats, survivor_cap=1.0)
            k, s = pred.key, pred.stats
        keys.append(k)
        st = merge_stats(st, s) if stats else None
    key = keys[0] if len(keys) == 1 else torch.cat(keys)
    idx, lab, dist = finalize(key, model.labels, 0, stream)
    return Prediction(idx, lab, dist, st, key)


def loocv_window(x: torch.Tensor, labels: torch.Tensor, windows, v: int = 5, q_begin: int = 0,
                 q_end: int | None = None, with_nn: bool = False, stats: bool = False,
                 stream=None):
    """S8: leave-one-out error counts per window (device int64 [nw]) and optional NN ids."""
    _series(x, "x")
    n, L = x.shape
    q_end = n if q_end is None else int(q_end)
    labels = labels.to(device=x.device, dtype=torch.int32).contiguous()
    win = (C.c_int32 * len(windows))(*[int(w) for w in windows])
    nw = len(windows)
    need = load().nndtw_loocv_workspace_bytes(n, L, q_begin, q_end)
    ws = torch.empty(need, dtype=torch.uint8, device=x.device)
    errors = torch.zeros(nw, dtype=torch.int64, device=x.device)
    nn = (torch.empty((nw, q_end - q_begin), dtype=torch.int32, device=x.device)
          if with_nn else None)
    st = Stats()
    _check(load().nndtw_loocv_window(_ptr(x), _ptr(labels), n, L, C.cast(win, C.c_void_p), nw,
                                     int(v), int(q_begin), q_end, _ptr(ws), ws.numel(),
                                     _ptr(errors), _ptr(nn), C.byref(st) if stats else None,
                                     _stream(stream)), "nndtw_loocv_window")
    return errors, nn, (st.as_dict() if stats else None)


class GraphedClassifier:
    """classify() for a fixed (model, nq), captured once into a CUDA graph and replayed: the
    ~25 launches of a call (bound, seeds, compaction, DTW, fp64 near-tie re-rank, decode)
    become one graph launch.  For launch-bound small problems (BJ:configs[0], [1]).

    `__call__(q)` copies q into the graph's static input and replays; the returned Prediction
    tensors are the graph's static outputs (overwritten by the next call -- clone to keep).
    Inputs are not NaN-checked inside the graph (check once with check_finite)."""

    def __init__(self, model: Model, nq: int):
        dev = model.t.device
        self.model = model
        self.q = torch.zeros((nq, model.L), dtype=torch.float32, device=dev)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        # the full workspace layout: a capped one needs a host check of its overflow word after
        # every call, which a graph cannot contain
        with torch.cuda.stream(side):  # warm-up: workspace, kernel attributes
            classify(model, self.q, check=False, survivor_cap=1.0)
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.pred = classify(model, self.q, check=False, survivor_cap=1.0)

    def __call__(self, q: torch.Tensor) -> Prediction:
        self.q.copy_(q, non_blocking=True)
        self.graph.replay()
        return self.pred


class GraphedLoocv:
    """loocv_window() over a fixed window list captured into one CUDA graph (101 windows x
    ~25 launches -> one graph launch).  `__call__()` replays and returns the device errors
    [nw] (static tensor, recomputed from zero on every replay)."""

    def __init__(self, x: torch.Tensor, labels: torch.Tensor, windows, v: int = 5):
        _series(x, "x")
        n, L = x.shape
        self.x = x
        self.labels = labels.to(device=x.device, dtype=torch.int32).contiguous()
        self.win = (C.c_int32 * len(windows))(*[int(w) for w in windows])
        self.nw = len(windows)
        self.v = int(v)
        need = load().nndtw_loocv_workspace_bytes(n, L, 0, n)
        self.ws = torch.empty(need, dtype=torch.uint8, device=x.device)
        self.errors = torch.zeros(self.nw, dtype=torch.int64, device=x.device)
        side = torch.cuda.Stream(device=x.device)
        side.wait_stream(torch.cuda.current_stream(x.device))
        with torch.cuda.stream(side):
            self._run()
        torch.cuda.current_stream(x.device).wait_stream(side)
        torch.cuda.synchronize(x.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._run()

    def _run(self):
        n, L = self.x.shape
        self.errors.zero_()
        _check(load().nndtw_loocv_window(_ptr(self.x), _ptr(self.labels), n, L,
                                         C.cast(self.win, C.c_void_p), self.nw, self.v, 0, n,
                                         _ptr(self.ws), self.ws.numel(), _ptr(self.errors),
                                         None, None, _stream()), "nndtw_loocv_window")

    def __call__(self) -> torch.Tensor:
        self.graph.replay()
        return self.errors


def launch_count() -> int:
    return int(load().nndtw_launch_count())
