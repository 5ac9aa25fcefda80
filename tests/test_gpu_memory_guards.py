"""Memory-safety checks of every C-ABI entry point without compute-sanitizer (closed on this
GPU pool, SURVEY.md §5 "race detection" asks for its equivalent):

* out-of-bounds WRITES: every output and workspace buffer sits between guard zones of 64 KiB
  filled with a sentinel pattern; after the call (and a synchronisation) the zones must be
  intact -- a kernel writing one element past its buffer, or a workspace carve-up overlapping
  the next region, changes them;
* reads of uninitialised workspace (initcheck's question): classify and LOOCV run with the
  workspace poisoned three ways (zero bytes, 0xFF bytes, random bytes); the answers must be
  bit-identical;
* races (racecheck's question, as far as results can show it): repeated calls give
  bit-identical keys, bounds and DTW values.
The debug build (NNDTW_DEBUG=1: device-side bounds asserts, a synchronisation and error check
after every launch) runs the same cases in tools/sanitize_cases.py."""
import numpy as np
import pytest

import datagen

from test_gpu_parity import T, dev  # noqa: F401

pytestmark = pytest.mark.gpu

GUARD = 16384  # 32-bit words = 64 KiB on each side
SENT = 0x7FBADBAD


class Guarded:
    """A device buffer of `n` elements of `dtype` between two sentinel-filled guard zones."""

    def __init__(self, n, dtype, dev, fill=None):
        import torch
        esz = torch.empty(0, dtype=dtype).element_size()
        nbytes = max(int(n), 1) * esz
        nwords = (nbytes + 3) // 4
        self.raw = torch.full((2 * GUARD + nwords,), SENT, dtype=torch.int32, device=dev)
        mid = self.raw[GUARD:GUARD + nwords]
        if fill is not None:
            mid.view(torch.uint8)[:].fill_(fill)
        self.t = mid.view(torch.uint8)[:nbytes].view(dtype)
        self.nwords = nwords

    def ptr(self):
        import ctypes as C
        return C.c_void_p(self.t.data_ptr())

    def intact(self):
        import torch
        torch.cuda.synchronize()
        g = self.raw[:GUARD], self.raw[GUARD + self.nwords:]
        return all(bool((x == SENT).all()) for x in g)


def _env(dev, X, w):
    from paper_1808_09617_b200 import nndtw
    return nndtw.envelopes(T(X, dev), w)


def test_guards_s1_s2_s4_entry_points(dev):
    import torch
    from paper_1808_09617_b200 import nndtw
    lib, p, st = nndtw.load(), nndtw._ptr, nndtw._stream()
    rng = np.random.default_rng(3)
    for L, w in ((31, 4), (300, 60), (512, 103), (2048, 2047)):
        n = 37
        X = T(datagen.random_series(rng, n, L, "walk"), dev)
        Q = T(datagen.random_series(rng, 13, L, "walk"), dev)
        U, Lo_ = Guarded(n * L, torch.float32, dev), Guarded(n * L, torch.float32, dev)
        kim = Guarded(n * 4, torch.int32, dev)
        assert lib.nndtw_envelopes(p(X), n, L, w, U.ptr(), Lo_.ptr(), kim.ptr(), st) == 0
        assert U.intact() and Lo_.intact() and kim.intact(), (L, w)
        qk = Guarded(13 * 4, torch.int32, dev)
        assert lib.nndtw_series_stats(p(Q), 13, L, qk.ptr(), st) == 0
        assert qk.intact()
        ldlb = n + 3  # a row stride larger than nt: nothing may land in the gaps either
        for flags in (0, 1, 2, 3):
            lb = Guarded(13 * ldlb, torch.float32, dev, fill=0xFF)
            assert lib.nndtw_lb_enhanced(p(Q), 13, qk.ptr(), p(X), U.ptr(), Lo_.ptr(), kim.ptr(),
                                         n, L, w, 5, flags, lb.ptr(), ldlb, st) == 0
            assert lb.intact(), (L, w, flags)
            gaps = lb.t.view(13, ldlb)[:, n:].contiguous().view(torch.int32)
            assert bool((gaps == -1).all()), "wrote into the ldlb gap"
        qU, qL, _ = nndtw.envelopes(Q, w)
        lb = Guarded(13 * ldlb, torch.float32, dev)
        assert lib.nndtw_lb_enhanced_symmetric(p(Q), p(qU), p(qL), qk.ptr(), 13, p(X), U.ptr(),
                                               Lo_.ptr(), kim.ptr(), n, L, w, 5, 1, lb.ptr(),
                                               ldlb, st) == 0
        assert lb.intact()
        for fn in ("nndtw_lb_improved", "nndtw_lb_enhanced_improved"):
            lb = Guarded(13 * ldlb, torch.float32, dev)
            args = [p(Q), 13, p(X), U.ptr(), Lo_.ptr(), n, L, w]
            if fn == "nndtw_lb_enhanced_improved":
                args.append(5)
            assert getattr(lib, fn)(*args, lb.ptr(), ldlb, st) == 0
            assert lb.intact(), (fn, L, w)
        if L <= 512:
            lb = Guarded(13 * ldlb, torch.float32, dev)
            assert lib.nndtw_lb_new(p(Q), 13, p(X), n, L, w, lb.ptr(), ldlb, st) == 0
            assert lb.intact()
        npairs = 29
        ia = T(rng.integers(0, 13, npairs).astype(np.int32), dev)
        ib = T(rng.integers(0, n, npairs).astype(np.int32), dev)
        out = Guarded(npairs, torch.float32, dev)
        assert lib.nndtw_dtw_batch(p(Q), p(X), p(ia), p(ib), npairs, L, w, None, out.ptr(),
                                   st) == 0
        assert out.intact(), (L, w)
        for ww in (0, min(w, 30)):
            out = Guarded(npairs, torch.float32, dev)
            assert lib.nndtw_dtw_batch(p(Q), p(X), p(ia), p(ib), npairs, L, ww, None,
                                       out.ptr(), st) == 0
            assert out.intact(), (L, ww)


def _classify_raw(dev, Tr, trl, Q, w, V, flags, ws_fill, self_offset=-1):
    import torch
    from paper_1808_09617_b200 import nndtw
    lib, p, st = nndtw.load(), nndtw._ptr, nndtw._stream()
    t = T(Tr, dev)
    U, Lo, kim = nndtw.envelopes(t, w)
    q = T(Q, dev)
    nq, L = Q.shape
    nt = Tr.shape[0]
    need = lib.nndtw_classify_workspace_bytes(nq, nt, L, w)
    ws = Guarded(need, torch.uint8, dev, fill=None if ws_fill == "random" else ws_fill)
    if ws_fill == "random":
        ws.t.copy_(torch.randint(0, 256, (need,), dtype=torch.uint8, device=dev))
    key = Guarded(nq, torch.int64, dev)
    stats = nndtw.Stats()
    import ctypes as C
    rc = lib.nndtw_classify(p(q), nq, p(t), p(U), p(Lo), p(kim), nt, 0, self_offset, L, w, V,
                            flags, ws.ptr(), need, key.ptr(), C.byref(stats), st)
    assert rc == 0, lib.nndtw_last_error()
    assert ws.intact() and key.intact()
    return key.t.cpu().numpy().copy(), stats.as_dict()


@pytest.mark.parametrize("stages", ["1", "2"])
@pytest.mark.parametrize("flags", [1, 1 | 128, 1 | 2, 1 | 4, 1 | 256, 1 | 512, 1 | 1024, 1 | 2048])
def test_classify_workspace_guards_and_poisoning(dev, monkeypatch, flags, stages):
    """All classify variants (EXACT with level counters, the Keogh / symmetric / LB_Improved /
    LB_New / enhanced+improved / no bound S2; the default cascade in one and in two stages):
    workspace and key guard zones intact, and the same keys with the workspace poisoned with
    zeros, 0xFF bytes and random bytes."""
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    ds = datagen.make_dataset(1, n_train=300, n_test=70)
    w = datagen.window_from_percent(20, 256)
    keys = [_classify_raw(dev, ds.train, ds.train_labels, ds.test, w, 5, flags, f)[0]
            for f in (0, 0xFF, "random")]
    assert np.array_equal(keys[0], keys[1]) and np.array_equal(keys[0], keys[2])


@pytest.mark.parametrize("stages", ["1", "2"])
def test_classify_ga_layout_guards_and_poisoning(dev, oracle_lib, monkeypatch, stages):
    """Config 2's band layout (L = 512, w = 103: R = 26, full warp, half-packed), whose survivor
    round reads the query rows from the padded copy in the workspace (GA variant, k_pad_rows):
    guard zones intact, the same keys under zero / 0xFF / random workspace poisoning, and the
    oracle's neighbours."""
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    ds = datagen.make_dataset(2, n_train=400, n_test=48)
    w = ds.cfg.windows()[0]
    assert w == 103
    runs = [_classify_raw(dev, ds.train, ds.train_labels, ds.test, w, 5, 1, f)
            for f in (0, 0xFF, "random")]
    keys = [r[0] for r in runs]
    assert np.array_equal(keys[0], keys[1]) and np.array_equal(keys[0], keys[2])
    assert runs[0][1]["dtw_calls"] > 0
    idx = (keys[0] & 0xFFFFFFFF).astype(np.int64)
    ridx, _ = oracle_lib.nn(ds.test, ds.train, w)[:2]
    assert np.array_equal(idx, ridx)


def test_loocv_workspace_guards_and_poisoning(dev):
    import torch
    from paper_1808_09617_b200 import nndtw
    lib, p, st = nndtw.load(), nndtw._ptr, nndtw._stream()
    ds = datagen.make_dataset(3, n_train=150)
    X, lab = T(ds.train, dev), T(ds.train_labels, dev)
    n, L = ds.train.shape
    wins = (0, 3, 30, 150, 299)
    import ctypes as C
    win = (C.c_int32 * len(wins))(*wins)
    res = []
    for fill in (0, 0xFF, "random"):
        need = lib.nndtw_loocv_workspace_bytes(n, L, 20, 130)
        ws = Guarded(need, torch.uint8, dev, fill=0 if fill == "random" else fill)
        if fill == "random":
            ws.t.copy_(torch.randint(0, 256, (need,), dtype=torch.uint8, device=dev))
        err = Guarded(len(wins), torch.int64, dev, fill=0)
        nn = Guarded(len(wins) * 110, torch.int32, dev)
        assert lib.nndtw_loocv_window(p(X), p(lab), n, L, C.cast(win, C.c_void_p), len(wins), 5,
                                      20, 130, ws.ptr(), need, err.ptr(), nn.ptr(), None, st) == 0
        assert ws.intact() and err.intact() and nn.intact()
        res.append((err.t.cpu().numpy().copy(), nn.t.cpu().numpy().copy()))
    for e, n_ in res[1:]:
        assert np.array_equal(e, res[0][0]) and np.array_equal(n_, res[0][1])


def test_sharded_refine_resolve_finalize_guards(dev):
    import torch
    from paper_1808_09617_b200 import nndtw
    lib, p, st = nndtw.load(), nndtw._ptr, nndtw._stream()
    ds = datagen.make_dataset(0)
    w = ds.cfg.windows()[0]
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    q = T(ds.test[:50], dev)
    key, ws, _ = nndtw.classify_keys(model, q, exact=False)
    f64 = Guarded(50, torch.int64, dev)
    assert lib.nndtw_classify_refine(p(ws), ws.numel(), p(q), 50, p(model.t), 100, 128, w, p(key),
                                     f64.ptr(), st) == 0
    assert f64.intact()
    out = Guarded(50, torch.int64, dev)
    assert lib.nndtw_classify_resolve(p(ws), ws.numel(), p(q), 50, p(model.t), 100, 128, w, 0,
                                      p(key), p(f64.t), out.ptr(), st) == 0
    assert out.intact()
    idx, lab, dist = (Guarded(50, torch.int64, dev), Guarded(50, torch.int32, dev),
                      Guarded(50, torch.float32, dev))
    assert lib.nndtw_finalize(p(out.t), 50, 1, p(model.labels), 100, idx.ptr(), lab.ptr(),
                              dist.ptr(), st) == 0
    assert idx.intact() and lab.intact() and dist.intact()
    s, c, m = (Guarded(1, torch.float64, dev, fill=0), Guarded(1, torch.int64, dev, fill=0),
               Guarded(1, torch.int32, dev, fill=0))
    d = torch.rand(1000, device=dev) + 0.5
    lbv = d * 0.5
    assert lib.nndtw_tightness(p(lbv), p(d), 1000, s.ptr(), c.ptr(), m.ptr(), st) == 0
    assert s.intact() and c.intact() and m.intact()
    bad = Guarded(1, torch.int32, dev, fill=0)
    assert lib.nndtw_check_finite(p(q), q.numel(), bad.ptr(), st) == 0
    assert bad.intact()


def test_repeated_calls_bit_identical(dev):
    """Races would show up as run-to-run differences: bounds, DTW values and NN keys of three
    identical calls are bit-identical (the survivor round's order and live best-so-far vary from
    run to run -- the answer must not)."""
    import torch
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(2, n_train=3000, n_test=200)
    t, q = T(ds.train, dev), T(ds.test, dev)
    w = 103
    U, Lo, kim = nndtw.envelopes(t, w)
    model = nndtw.Model(t, T(ds.train_labels, dev), w, 5)
    ref = None
    for _ in range(3):
        lb = nndtw.lb_enhanced(q, t, U, Lo, w, 5, with_kim=True, tkim=kim)
        ia = torch.arange(200, device=dev, dtype=torch.int32)
        d = nndtw.dtw_batch(q, t, w, ia, ia * 7)
        k, _, _ = nndtw.classify_keys(model, q, exact=True)
        e2, e3, e4 = nndtw.envelopes(t, w)
        cur = [x.cpu().numpy().copy() for x in (lb, d, k, e2, e3, e4)]
        if ref is None:
            ref = cur
        for a, b in zip(ref, cur):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
