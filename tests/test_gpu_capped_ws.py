"""Capped classify workspace (nndtw_classify_workspace_bytes_capped / nndtw_classify_overflowed):
room for a fraction of the (query, train) pairs as survivors and two-stage list entries instead
of all of them.  A call that needs more must report the overflow (its keys are invalid), never
write outside the workspace, and nndtw.classify must then rerun it with the full layout -- the
answer is the fp64 oracle's either way (tests/golden, every query)."""
import numpy as np
import pytest
import torch

import datagen

from test_gpu_golden import _compare, dataset, golden
from test_gpu_parity import T, dev  # noqa: F401

pytestmark = pytest.mark.gpu


def _model(dev, ds, w, V=5):
    from paper_1808_09617_b200 import nndtw
    return nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, V)


@pytest.mark.parametrize("stages", ["1", "2"])
def test_overflow_is_reported_and_guarded(dev, monkeypatch, stages):
    """A capacity far below the survivor count: the overflow word is set, and the workspace
    bytes past the layout (poisoned) are untouched -- the clamped lists keep every reader and
    writer inside it."""
    from paper_1808_09617_b200 import nndtw
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    ds = dataset(1)
    w = datagen.window_from_percent(20, 256)
    model = _model(dev, ds, w)
    q = T(ds.test, dev)
    nq, nt = q.shape[0], model.t.shape[0]
    lib = nndtw.load()
    cap = 2 * nq + 2  # the smallest capacity (the seed rounds)
    need = lib.nndtw_classify_workspace_bytes_capped(nq, nt, model.L, w, cap)
    full = lib.nndtw_classify_workspace_bytes(nq, nt, model.L, w)
    assert need < full
    guard = 1 << 20
    buf = torch.full((need + guard,), 0x5A, dtype=torch.uint8, device=dev)
    ws = buf[:need]
    key2 = torch.empty(nq, dtype=torch.int64, device=dev)
    flags = nndtw.NNDTW_CLASSIFY_EXACT
    nndtw._check(lib.nndtw_classify(nndtw._ptr(q), nq, nndtw._ptr(model.t), nndtw._ptr(model.U),
                                    nndtw._ptr(model.Lo), nndtw._ptr(model.kim), nt, 0, -1,
                                    model.L, w, model.v, flags, nndtw._ptr(ws), ws.numel(),
                                    nndtw._ptr(key2), None, nndtw._stream(None)), "classify")
    assert nndtw.classify_overflowed(model, nq, ws)
    torch.cuda.synchronize()
    assert bool((buf[need:] == 0x5A).all()), "write past the capped workspace"


@pytest.mark.parametrize("stages", ["1", "2"])
def test_capped_classify_reruns_and_matches_oracle(dev, monkeypatch, stages):
    """nndtw.classify with a capacity too small for config 1's survivors: the rerun with the
    full layout gives every query's oracle answer."""
    from paper_1808_09617_b200 import nndtw
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(20, 256)
    model = _model(dev, ds, w)
    p = nndtw.classify(model, T(ds.test, dev), survivor_cap=1e-6, stats=True)
    _compare(p.idx.cpu().numpy(), p.label.cpu().numpy(), p.dist.cpu().numpy(),
             g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"], f"capped, stages={stages}")
    assert p.stats["survivors"] > 2 * ds.test.shape[0] + 2  # (the capacity was exceeded)


@pytest.mark.parametrize("stages", ["1", "2"])
def test_capped_classify_without_overflow(dev, monkeypatch, stages):
    """The default capacity holds config 1's survivors: no overflow, the oracle's answers, and
    a workspace well below the full layout's."""
    from paper_1808_09617_b200 import nndtw
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(10, 256)
    model = _model(dev, ds, w)
    q = T(ds.test, dev)
    nq, nt = q.shape[0], model.t.shape[0]
    mp = int(nndtw.SURVIVOR_CAP * nq * nt) + 1
    key, ws, st = nndtw.classify_keys(model, q, max_pairs=mp, stats=True)
    assert not nndtw.classify_overflowed(model, nq, ws)
    assert st["survivors"] <= mp
    lib = nndtw.load()
    assert lib.nndtw_classify_workspace_bytes_capped(nq, nt, model.L, w, mp) < \
        0.5 * lib.nndtw_classify_workspace_bytes(nq, nt, model.L, w)
    idx, lab, dist = nndtw.finalize(key, model.labels)
    _compare(idx.cpu().numpy(), lab.cpu().numpy(), dist.cpu().numpy(),
             g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"], f"capped, stages={stages}")


def test_graphed_classifier_uses_full_layout(dev):
    """The CUDA-graph replay cannot check the overflow word on the host: it keeps the full
    layout and still matches the oracle."""
    from paper_1808_09617_b200 import nndtw
    g = golden(0)
    ds = dataset(0)
    w = int(g["w"])
    model = _model(dev, ds, w)
    gc = nndtw.GraphedClassifier(model, ds.test.shape[0])
    p = gc(T(ds.test, dev))
    _compare(p.idx.cpu().numpy(), p.label.cpu().numpy(), p.dist.cpu().numpy(),
             g["idx"], g["label"], g["dist"], "graphed config 0")
