"""S4 band-limited pass: wide windows run the survivors first
in a band of window wb < w with a check of the band-edge cells; items whose edges come within
the threshold are rerun with the full window.  The answer must be the full-window one, i.e.
the fp64 oracle's (tests/golden, every query) -- with the default wb, with forced narrow bands
that send many items to the full-window pass, and when the appended items do not fit in the
item array (every survivor is rerun)."""
import numpy as np
import pytest

import datagen

from test_gpu_golden import _compare, dataset, golden
from test_gpu_parity import T, dev  # noqa: F401

pytestmark = pytest.mark.gpu


def _run(dev, ds, w, max_pairs=None, V=5):
    from paper_1808_09617_b200 import nndtw
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, V)
    q = T(ds.test, dev)
    key, ws, st = nndtw.classify_keys(model, q, stats=True, max_pairs=max_pairs)
    assert not nndtw.classify_overflowed(model, q.shape[0], ws)
    idx, lab, dist = nndtw.finalize(key, model.labels)
    return idx.cpu().numpy(), lab.cpu().numpy(), dist.cpu().numpy(), st


@pytest.mark.parametrize("p", [20, 50, 100])
@pytest.mark.parametrize("adapt", ["-1", "12", "25", "51"])
def test_adapt_config1_matches_oracle(dev, monkeypatch, p, adapt):
    """(w = 255 is the full window: the row-strip kernel, no band-limited pass; w = 52 runs it
    only when forced, wb < w)"""
    monkeypatch.setenv("NNDTW_ADAPT", adapt)
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(p, 256)
    idx, lab, dist, st = _run(dev, ds, w)
    _compare(idx, lab, dist, g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"],
             f"NNDTW_ADAPT={adapt} w={w}")
    if adapt == "12" and p == 50:  # a 25-offset band on a 257-offset window: many fall back
        assert st["dtw_fallback"] > 0, st
    if p == 100:
        assert st["dtw_fallback"] == 0, st


def test_adapt_off_and_on_same_counts_of_work(dev, monkeypatch):
    """Off, the survivor round never falls back; on, it does less DP work for the same answer."""
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(50, 256)
    monkeypatch.setenv("NNDTW_ADAPT", "0")
    i0, l0, d0, s0 = _run(dev, ds, w)
    monkeypatch.setenv("NNDTW_ADAPT", "-1")
    i1, l1, d1, s1 = _run(dev, ds, w)
    assert s0["dtw_fallback"] == 0
    assert s1["cells"] < s0["cells"], (s0, s1)
    assert np.array_equal(i0, i1) and np.array_equal(l0, l1)
    _compare(i1, l1, d1, g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"], "adapt on")


def test_adapt_fallback_items_do_not_fit(dev, monkeypatch):
    """A capped workspace with room for barely more than the survivors: the appended items do
    not all fit, so the full-window pass reruns every survivor -- still the oracle's answer."""
    monkeypatch.setenv("NNDTW_ADAPT", "12")
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(50, 256)
    _, _, _, st = _run(dev, ds, w)
    assert st["dtw_fallback"] > 64, st
    idx, lab, dist, st2 = _run(dev, ds, w, max_pairs=st["survivors"] + 16)
    _compare(idx, lab, dist, g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"], "no room")
    assert st2["dtw_fallback"] > 64, st2


@pytest.mark.parametrize("L,w,shift", [(512, 103, 30), (512, 103, 70), (512, 103, 100),
                                         (1024, 1023, 60), (1024, 1023, 160), (1024, 1023, 300)])
def test_adapt_warped_neighbours_fall_back_exactly(dev, oracle_lib, L, w, shift):
    """Adversarial for the band edge: every query is a train series shifted by `shift` samples,
    so for shift > wb (w = 103: wb = 51, the band kernel's fallback; the full window at L = 1024:
    wb = 103, the row-strip kernel's fallback) its nearest neighbour's warping path leaves the
    band -- the edge check must send those items to the full window, and every answer must be
    the fp64 oracle's (exhaustive)."""
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(shift)
    ns, nq = 32, 24
    wb_ = nndtw.load().nndtw_band_limited_window(L, w)
    assert wb_ == (51 if w == 103 else 103)
    walk = np.cumsum(rng.standard_normal((ns, L + 2 * shift + 4)), axis=1)
    # three noisy variants of every source (offsets 0, 1, 2): near-ties the survivor round must
    # evaluate in full, all of them warped by about `shift` against their query
    T_ = np.concatenate([walk[:, shift + o:shift + o + L] + 0.05 * rng.standard_normal((ns, L))
                         for o in (0, 1, 2)])
    nt = T_.shape[0]
    src = rng.choice(ns, nq, replace=False)
    Q_ = walk[src, 2 * shift + 1:2 * shift + 1 + L] + 0.05 * rng.standard_normal((nq, L))
    z = lambda x: ((x - x.mean(1, keepdims=True)) / x.std(1, keepdims=True)).astype(np.float32)
    T_, Q_ = z(T_), z(Q_)
    labels = (np.arange(nt) % 5).astype(np.int32)
    model = nndtw.Model(T(T_, dev), T(labels, dev), w, 5)
    key, ws, st = nndtw.classify_keys(model, T(Q_, dev), stats=True)
    idx, lab, dist = nndtw.finalize(key, model.labels)
    ridx, rdist = oracle_lib.nn(Q_, T_, w, mode="exhaustive")
    idx = idx.cpu().numpy()
    assert np.array_equal(idx, ridx), (shift, np.nonzero(idx != ridx)[0][:8])
    d = dist.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(d - rdist) <= 1e-5 * rdist + 1e-30)
    if shift > wb_:
        assert st["dtw_fallback"] > 0, st
    if shift > wb_ and st["dtw_fallback"] > 1:
        # no room for the appended items (a capped workspace one pair above the survivors):
        # the full-window pass (band or row-strip kernel) reruns every survivor -- same answer
        key2, ws2, st2 = nndtw.classify_keys(model, T(Q_, dev), stats=True,
                                             max_pairs=st["survivors"] + 1)
        assert not nndtw.classify_overflowed(model, nq, ws2)
        idx2, _, dist2 = nndtw.finalize(key2, model.labels)
        assert np.array_equal(idx2.cpu().numpy(), ridx)
        assert np.all(np.abs(dist2.cpu().numpy().astype(np.float64) - rdist) <=
                      1e-5 * rdist + 1e-30)
