"""The two-stage S2 (lb_sparse.cu: LB_Kim + Algorithm 1's bands for every pair, a seed round, the
LB_Keogh bridge only for the pairs the partial cascade keeps -- Algorithm 1's line-12 test,
P:535 -- and a second seed round) forced on with NNDTW_S2_STAGES=2 on inputs where the library
would pick one stage, so that every query of the small golden configs, the tie grids, LOOCV
and the level counters run through it.  The default (size-gated) choice runs it on config 2,
whose every query tests/test_gpu_golden.py checks."""
import numpy as np
import pytest

import datagen

from test_gpu_golden import _compare, dataset, golden
from test_gpu_parity import T, _check_nn, _classify, dev  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.fixture
def two_stage(monkeypatch):
    monkeypatch.setenv("NNDTW_S2_STAGES", "2")


def test_two_stage_golden_configs_0_1(dev, two_stage):
    from paper_1808_09617_b200 import nndtw
    g0, ds0 = golden(0), dataset(0)
    model = nndtw.Model(T(ds0.train, dev), T(ds0.train_labels, dev), int(g0["w"]), 5)
    p = nndtw.classify(model, T(ds0.test, dev), stats=True)
    assert p.stats["bridge_pairs"] < p.stats["lb_pairs"]  # the two-stage path ran
    _compare(p.idx.cpu().numpy(), p.label.cpu().numpy(), p.dist.cpu().numpy(), g0["idx"],
             g0["label"], g0["dist"], "two-stage config 0")
    g1, ds1 = golden(1), dataset(1)
    for pct in (1, 10, 20, 50, 100):
        w = datagen.window_from_percent(pct, 256)
        for V in (1, 5, 8):
            model = nndtw.Model(T(ds1.train, dev), T(ds1.train_labels, dev), w, V)
            p = nndtw.classify(model, T(ds1.test, dev))
            _compare(p.idx.cpu().numpy(), p.label.cpu().numpy(), p.dist.cpu().numpy(),
                     g1[f"idx_w{w}"], g1[f"label_w{w}"], g1[f"dist_w{w}"],
                     f"two-stage config 1 w={w} V={V}")


@pytest.mark.parametrize("kind,L,w,V", [("int", 8, 2, 3), ("int", 16, 0, 5), ("int", 33, 32, 4),
                                        ("walk", 2, 0, 1), ("walk", 3, 1, 5), ("const", 12, 3, 2),
                                        ("walk", 130, 129, 16), ("int", 64, 5, 1),
                                        ("walk", 300, 30, 5), ("walk", 1000, 100, 8),
                                        ("walk", 128, 40, 16), ("int", 36, 35, 16),
                                        ("walk", 4, 3, 2), ("int", 24, 6, 12)])
def test_two_stage_ties_and_shapes(dev, oracle_lib, two_stage, kind, L, w, V):
    """Exact ties (integer grids, duplicates before and after), constant series, every L mod 4
    (the sparse kernel's register and scalar row paths), the V limits of the lane bands and of
    the head/tail copies (nb = 16: one query per copy instruction; the ring smaller than the
    head/tail area at L <= 128)."""
    rng = np.random.default_rng(L * 37 + w)
    Tr = datagen.random_series(rng, 257, L, kind)
    Tr[200:210] = Tr[17]
    Tr[3] = Tr[250]
    Q = datagen.random_series(rng, 61, L, kind)
    Q[0] = Tr[17]
    trl = rng.integers(0, 4, size=257).astype(np.int32)
    idx, lab, dist, st = _classify(dev, Tr, trl, Q, w, V, stats=True)
    _check_nn(oracle_lib, Tr, trl, Q, w, idx, lab, dist)


def test_two_stage_loocv(dev, oracle_lib, two_stage):
    """Leave-one-out (the self pair is NaN in stage A and never listed) with the previous
    window's neighbour as an extra first-round seed."""
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(3, n_train=240)
    X, lab = ds.train, ds.train_labels
    windows = [datagen.window_from_percent(p, 300) for p in (0, 1, 2, 5, 10, 30, 70, 100)]
    err, nn, _ = nndtw.loocv_window(T(X, dev), T(lab, dev), windows, v=5, with_nn=True)
    rerr, rnn = oracle_lib.loocv(X, lab, windows, V=5, mode="pruned")
    assert np.array_equal(nn.cpu().numpy(), rnn.astype(np.int32))
    assert np.array_equal(err.cpu().numpy(), rerr)


def test_two_stage_long_rows_scalar_path(dev, oracle_lib, two_stage):
    """L = 2048, full window, V = 8 (config 4's shape, the sparse kernel's scalar row path)."""
    ds = datagen.make_dataset(4, n_train=300, n_test=12)
    w = ds.cfg.windows()[0]
    idx, lab, dist, st = _classify(dev, ds.train, ds.train_labels, ds.test, w, 8, stats=True)
    _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test, w, idx, lab, dist)


@pytest.mark.parametrize("ed", ["0", "1"])
def test_two_stage_level_counters(dev, two_stage, monkeypatch, ed):
    """The level counters partition the pairs under the two-stage path too (excluded seeds: the
    full-cascade argmin of every query, and with the Euclidean first seed that one too where it
    differs), and the bridge ran on fewer pairs than the bound."""
    from paper_1808_09617_b200 import nndtw
    monkeypatch.setenv("NNDTW_ED_SEED", ed)
    ds = datagen.make_dataset(1)
    w = datagen.window_from_percent(10, 256)
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    st = nndtw.classify(model, T(ds.test[:300], dev), stats=True, level_stats=True).stats
    pruned = st["pruned_kim"] + st["pruned_bands"] + st["pruned_keogh"]
    if ed == "0":
        assert pruned + st["survivors"] + 300 == st["lb_pairs"], st
    else:
        assert st["lb_pairs"] - 600 <= pruned + st["survivors"] <= st["lb_pairs"] - 300, st
    assert 0 < st["bridge_pairs"] < st["lb_pairs"]
    # every pair kept after stage A had its bridge computed: the final bridge-level prunes and
    # the survivors are a subset of the bridge pairs
    assert st["pruned_keogh"] + st["survivors"] <= st["bridge_pairs"]
    assert st["ms_lb_bridge"] > 0.0


def test_two_stage_sharded_phases(dev, two_stage):
    """The seed phase (stages A and B, both seed rounds) and the search phase of a sharded call
    give the same key as one call (shard of the whole set, one rank)."""
    import torch
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(1)
    w = datagen.window_from_percent(20, 256)
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    q = T(ds.test[:200], dev)
    k1, _, _ = nndtw.classify_keys(model, q, exact=False)
    ks, ws, _ = nndtw.classify_keys(model, q, exact=False, phase="seed")
    k2, _, _ = nndtw.classify_keys(model, q, exact=False, phase="search", key=ks.clone(), ws=ws)
    assert torch.equal(k1, k2)


@pytest.mark.parametrize("nq,nt,L,kind", [(1, 1, 64, "walk"), (1, 500, 128, "walk"),
                                          (40, 1, 64, "walk"), (33, 70, 96, "int"),
                                          (65, 3, 256, "const"), (100, 90, 512, "walk")])
def test_two_stage_degenerate_sizes(dev, oracle_lib, two_stage, nq, nt, L, kind):
    """One query, one train series, 32k+1 queries per list (a one-entry batch after full ones),
    a list of every query on every series (constant series: every pair ties and survives)."""
    rng = np.random.default_rng(nq * 1000 + nt)
    Tr = datagen.random_series(rng, nt, L, kind)
    Q = datagen.random_series(rng, nq, L, kind)
    trl = rng.integers(0, 3, size=nt).astype(np.int32)
    w = max(1, L // 10)
    idx, lab, dist, st = _classify(dev, Tr, trl, Q, w, 5, stats=True)
    _check_nn(oracle_lib, Tr, trl, Q, w, idx, lab, dist)
    assert 0 <= st["bridge_pairs"] <= nq * nt
