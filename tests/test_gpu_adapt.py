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
