"""Full-size parity on BASELINE.json configs 0-4: EVERY query's 1-NN (index, label, distance)
and config 3's per-window leave-one-out neighbours and error counts, against the fp64
oracle's answers stored in tests/golden/cfg{k}.npz.

Those files are written by tests/golden/make_golden.py, which imports only oracle/ and datagen.py
(no value comes from the CUDA path).  Bar (north_star): indices and labels bit-exact, squared
distances within relative 1e-5; pruning is lossless by Theorem 2, so the pruned
GPU search must return the exact 1-NN with ties to the lowest index (reading C13).

The product calls are the ones bench.py times: nndtw.Model + nndtw.classify (S1-S7 on one
GPU), nndtw.loocv_window for S8, and dist.classify_sharded on a one-rank NCCL group for the
S6 path that bench.py runs under torchrun."""
import os
import socket

import numpy as np
import pytest

import datagen

from test_gpu_parity import T, assert_rel, dev  # noqa: F401

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(c):
    f = os.path.join(GOLDEN, f"cfg{c}.npz")
    if not os.path.exists(f):
        pytest.fail(f"{f} missing: run tests/golden/make_golden.py")
    return np.load(f)


_DS = {}


def dataset(c):
    if c not in _DS:
        _DS[c] = datagen.make_dataset(c)
    return _DS[c]


def _classify(dev, ds, w, V, stats_out=None, **kw):
    from paper_1808_09617_b200 import nndtw
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, V, **kw)
    p = nndtw.classify(model, T(ds.test, dev), stats=stats_out is not None)
    if stats_out is not None:
        stats_out.update(p.stats)
    return p.idx.cpu().numpy(), p.label.cpu().numpy(), p.dist.cpu().numpy()


def _compare(idx, lab, dist, ridx, rlab, rdist, what):
    bad = np.nonzero(idx != ridx)[0]
    assert bad.size == 0, f"{what}: {bad.size} NN index mismatches, first {bad[:8]}"
    assert np.array_equal(lab, rlab), what
    assert_rel(dist, rdist, what=what)


@pytest.mark.parametrize("c", [0, 2, 4])
def test_golden_classify_every_query(dev, c):
    g = golden(c)
    ds = dataset(c)
    w = int(g["w"])
    assert w == ds.cfg.windows()[0]
    V = int(g["V"]) if "V" in g else 5
    st = {}
    idx, lab, dist = _classify(dev, ds, w, V, stats_out=st)
    assert idx.shape[0] == ds.test.shape[0] == g["idx"].shape[0]
    _compare(idx, lab, dist, g["idx"], g["label"], g["dist"], f"config {c}")
    if c == 2:  # the size gate runs the default cascade in two stages here
        assert 0 < st["bridge_pairs"] < st["lb_pairs"], st


@pytest.mark.parametrize("p", [1, 10, 20, 50, 100])
def test_golden_config1_every_query_every_V(dev, p):
    """BJ:configs[1]: all 1000 queries at each window of the grid and each V of the grid (the
    bound changes, the answer must not)."""
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(p, 256)
    for V in ds.cfg.Vs:
        idx, lab, dist = _classify(dev, ds, w, V)
        _compare(idx, lab, dist, g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"],
                 f"config 1 w={w} V={V}")


def test_golden_config1_other_bounds_same_answer(dev):
    """The LB_Keogh cascade and the symmetric bound prune differently; the answer is the same."""
    g = golden(1)
    ds = dataset(1)
    w = datagen.window_from_percent(20, 256)
    for kw in ({"bound": "keogh"}, {"symmetric": True}):
        idx, lab, dist = _classify(dev, ds, w, 5, **kw)
        _compare(idx, lab, dist, g[f"idx_w{w}"], g[f"label_w{w}"], g[f"dist_w{w}"], str(kw))


def test_golden_config3_loocv_all_windows(dev):
    """BJ:configs[3]: 2000 series, all 101 windows (reading C17): every held-out
    series' neighbour in every window and the exact error counts."""
    from paper_1808_09617_b200 import nndtw
    from paper_1808_09617_b200.dist import best_window
    g = golden(3)
    ds = dataset(3)
    wins = ds.cfg.windows()
    assert list(g["windows"]) == wins
    err, nn, _ = nndtw.loocv_window(T(ds.train, dev), T(ds.train_labels, dev), wins, v=5,
                                    with_nn=True)
    nn = nn.cpu().numpy()
    for p in range(len(wins)):
        bad = np.nonzero(nn[p] != g["nn"][p])[0]
        assert bad.size == 0, f"window {wins[p]}: {bad.size} mismatches, first {bad[:8]}"
    assert np.array_equal(err.cpu().numpy(), g["errors"])
    assert best_window(err.cpu().tolist(), wins) == best_window(g["errors"].tolist(), wins)


def test_golden_config3_graphed_loocv(dev):
    """The CUDA-graph replay of the 101-window search gives the same counts (twice)."""
    from paper_1808_09617_b200 import nndtw
    g = golden(3)
    ds = dataset(3)
    gl = nndtw.GraphedLoocv(T(ds.train, dev), T(ds.train_labels, dev), ds.cfg.windows(), v=5)
    for _ in range(2):
        assert np.array_equal(gl().cpu().numpy(), g["errors"])


# ---------------------------------------------------------------- S6 on the product path
@pytest.fixture(scope="module")
def nccl_world1(dev):
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=dev)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("stages", ["1", "2"])
@pytest.mark.parametrize("split", [False, True])
@pytest.mark.parametrize("c,p", [(0, 10), (1, 10), (1, 100)])
def test_golden_classify_sharded_nccl(dev, nccl_world1, monkeypatch, stages, split, c, p):
    """dist.classify_sharded -- the two-phase seed exchange, the int64 MIN all-reduces of the
    fp32 keys, the fp64 near-tie keys and the resolved indices -- over a real NCCL group (one
    rank), on every query of configs 0 and 1, against the oracle; S2 in one and in two stages."""
    monkeypatch.setenv("NNDTW_S2_STAGES", stages)
    from paper_1808_09617_b200 import nndtw
    from paper_1808_09617_b200.dist import classify_sharded
    g = golden(c)
    ds = dataset(c)
    w = datagen.window_from_percent(p, ds.cfg.L)
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    pred = classify_sharded(model, T(ds.test, dev), T(ds.train_labels, dev), split=split)
    sfx = "" if c == 0 else f"_w{w}"
    _compare(pred.idx.cpu().numpy(), pred.label.cpu().numpy(), pred.dist.cpu().numpy(),
             g["idx" + sfx], g["label" + sfx], g["dist" + sfx], f"sharded config {c} w={w}")


def test_bench_sharded_path_runs(dev):
    """bench.py --sharded (the torchrun code path at N=1: NCCL group, classify_sharded) exits 0
    and prints a JSON line, so the multi-GPU launch cannot rot before an 8-GPU node runs it."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--sharded", "--config",
                        "1", "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--no-e2e"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and "x1" in line["config"]["parallelism"]
