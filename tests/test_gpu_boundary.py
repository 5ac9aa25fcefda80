"""Boundary details of include/nndtw.h on the GPU: per-level prune counters (P:299-304,
P:499-503), stage times, the input-magnitude precondition, the index range of the shard
combine, degenerate LOOCV, and the band layouts only reachable at particular windows."""
import ctypes as C

import numpy as np
import pytest

import datagen

from test_gpu_parity import T, _check_nn, _classify, assert_rel, dev  # noqa: F401

pytestmark = pytest.mark.gpu


def _model(dev, Tr, trl, w, V, **kw):
    from paper_1808_09617_b200 import nndtw
    return nndtw.Model(T(Tr, dev), T(trl, dev), w, V, **kw)


@pytest.mark.parametrize("bound", ["enhanced", "keogh", "symmetric"])
def test_level_counters_partition_the_pairs(dev, oracle_lib, bound):
    """pruned_kim + pruned_bands + pruned_keogh + survivors + seeds = lb_pairs, the counters are
    -1 unless asked for, and the answer is unchanged."""
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(1)
    w = datagen.window_from_percent(10, 256)
    kw = {"bound": "keogh"} if bound == "keogh" else ({"symmetric": True}
                                                      if bound == "symmetric" else {})
    model = _model(dev, ds.train, ds.train_labels, w, 5, **kw)
    q = T(ds.test[:200], dev)
    p0 = nndtw.classify(model, q, stats=True)
    assert p0.stats["pruned_kim"] == -1 and p0.stats["pruned_keogh"] == -1
    p1 = nndtw.classify(model, q, stats=True, level_stats=True)
    st = p1.stats
    assert np.array_equal(p0.idx.cpu().numpy(), p1.idx.cpu().numpy())
    pruned = st["pruned_kim"] + st["pruned_bands"] + st["pruned_keogh"]
    assert min(st["pruned_kim"], st["pruned_bands"], st["pruned_keogh"]) >= 0
    # one seed item per query here (the argmin-LB candidate)
    assert pruned + st["survivors"] + q.shape[0] == st["lb_pairs"], st
    if bound == "keogh":
        assert st["pruned_bands"] == 0     # no band stage in the LB_Keogh cascade
    else:
        assert st["pruned_bands"] > 0      # the V = 5 bands do prune on config-1 data
    assert pruned > 0.5 * st["lb_pairs"]
    assert st["ms_envelopes"] > 0.0 and st["ms_lb"] > 0.0 and st["ms_dtw"] > 0.0


def test_level_counters_against_oracle_levels(dev, oracle_lib):
    """Each pair's level recomputed in fp64 from the oracle's Kim and Algorithm-1 values against
    the GPU's seeded threshold (the DTW of the argmin-LB candidate, from the oracle), on pairs
    that are not within 1e-4 of the threshold."""
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(0)
    w = ds.cfg.windows()[0]
    V = 5
    Tr, Q = ds.train, ds.test[:40]
    model = _model(dev, Tr, ds.train_labels, w, V)
    pred = nndtw.classify(model, T(Q, dev), stats=True, level_stats=True)
    st = pred.stats
    U, Lo = oracle_lib.envelopes(Tr, w)
    cnt = np.zeros(3, np.int64)
    ambiguous = 0
    for i, a in enumerate(Q):
        full = np.array([oracle_lib.lb_cascade(a, b, U[j], Lo[j], w, V) for j, b in enumerate(Tr)])
        s1 = int(np.lexsort((np.arange(len(full)), full))[0])   # argmin, lowest index
        thr = oracle_lib.dtw(a, Tr[s1], w)
        inf = np.full(Q.shape[1], np.inf, np.float32)
        for j, b in enumerate(Tr):
            if j == s1:
                continue
            kim = oracle_lib.lb_kim_sum(a, b)
            # boundary terms + bands of Algorithm 1 alone: the bridge vanishes against the
            # envelope (+inf, -inf)
            band, _ = oracle_lib.lb_enhanced(a, b, inf, -inf, w, V)
            if min(abs(v - thr) for v in (kim, band, full[j])) <= 1e-4 * thr:
                ambiguous += 1
                continue
            if kim > thr:
                cnt[0] += 1
            elif full[j] > thr:
                cnt[1 if band > thr else 2] += 1
    got = np.array([st["pruned_kim"], st["pruned_bands"], st["pruned_keogh"]])
    assert np.all(np.abs(got - cnt) <= ambiguous), (got, cnt, ambiguous)
    assert ambiguous < 0.01 * len(Q) * len(Tr)


def test_magnitude_precondition(dev):
    from paper_1808_09617_b200 import nndtw
    x = np.zeros((3, 16), np.float32)
    assert nndtw.check_finite(T(x, dev))
    x[1, 5] = 2.0 ** 35
    assert nndtw.check_finite(T(x, dev))
    x[2, 7] = -(2.0 ** 36)
    assert not nndtw.check_finite(T(x, dev))
    with pytest.raises(nndtw.NNDTWError):
        _model(dev, x, np.zeros(3, np.int32), 3, 5)


def test_large_inputs_below_the_bound(dev, oracle_lib):
    """|x| up to 2^30: the kernels' +-2^64*k pads still give +inf out of the matrix."""
    rng = np.random.default_rng(11)
    A = (datagen.random_series(rng, 6, 100, "normal") * 2.0 ** 30).astype(np.float32)
    B = (datagen.random_series(rng, 6, 100, "normal") * 2.0 ** 30).astype(np.float32)
    from paper_1808_09617_b200 import nndtw
    for w in (0, 3, 30, 99):
        out = nndtw.dtw_batch(T(A, dev), T(B, dev), w).cpu().numpy()
        ref = np.array([oracle_lib.dtw(A[p], B[p], w) for p in range(6)])
        assert_rel(out, ref, what=f"w={w}")


def test_index_range_of_the_shard_combine(dev):
    """index_base + nt must stay below 2^31 (format-1 keys put the index in the high half of a
    signed int64)."""
    import torch
    from paper_1808_09617_b200 import nndtw
    lib = nndtw.load()
    x = T(datagen.random_series(np.random.default_rng(2), 4, 32, "walk"), dev)
    model = nndtw.Model(x, torch.zeros(4, dtype=torch.int32, device=dev), 3, 5)
    ws = model.workspace(4)
    key = torch.empty(4, dtype=torch.int64, device=dev)
    p = nndtw._ptr
    args = lambda base: (p(x), 4, p(x), p(model.U), p(model.Lo), p(model.kim), 4, base, -1, 32,  # noqa: E731
                         3, 5, 1, p(ws), ws.numel(), p(key), None, nndtw._stream())
    assert lib.nndtw_classify(*args(2 ** 31 - 5)) == 0
    assert lib.nndtw_classify(*args(2 ** 31 - 4)) == 8   # NNDTW_E_INDEX


def test_loocv_single_series(dev, oracle_lib):
    """n = 1: no other series, so no neighbour (-1) and one error; the held-out series is never
    its own neighbour (its bound is excluded from the seed and from the survivors)."""
    from paper_1808_09617_b200 import nndtw
    x = datagen.random_series(np.random.default_rng(4), 1, 40, "walk")
    lab = np.array([3], np.int32)
    err, nn, _ = nndtw.loocv_window(T(x, dev), T(lab, dev), [0, 4, 39], v=5, with_nn=True)
    rerr, rnn = oracle_lib.loocv(x, lab, [0, 4, 39], V=5)
    assert err.cpu().numpy().tolist() == [1, 1, 1] == rerr.tolist()
    assert (nn.cpu().numpy() == -1).all() and (rnn == -1).all()


def test_loocv_two_series(dev, oracle_lib):
    from paper_1808_09617_b200 import nndtw
    x = datagen.random_series(np.random.default_rng(5), 2, 40, "walk")
    lab = np.array([1, 2], np.int32)
    err, nn, _ = nndtw.loocv_window(T(x, dev), T(lab, dev), [0, 4, 39], v=5, with_nn=True)
    rerr, rnn = oracle_lib.loocv(x, lab, [0, 4, 39], V=5)
    assert np.array_equal(err.cpu().numpy(), rerr)
    assert np.array_equal(nn.cpu().numpy(), rnn.astype(np.int32))


def test_band_r32_layout(dev, oracle_lib):
    """2w+2 = 1024 (w = 511): the aligned R = 32, G = 32 band layout is the only one that fits;
    it must run (not the masked strip fallback) and match the oracle."""
    from paper_1808_09617_b200 import nndtw
    assert nndtw.load().nndtw_dtw_kernel_name(1024, 511) == b"k_dtw_band"
    rng = np.random.default_rng(511)
    A = datagen.random_series(rng, 5, 1024, "walk")
    B = datagen.random_series(rng, 5, 1024, "walk")
    out = nndtw.dtw_batch(T(A, dev), T(B, dev), 511).cpu().numpy()
    ref = np.array([oracle_lib.dtw(A[p], B[p], 511) for p in range(5)])
    assert_rel(out, ref, what="w=511")


def test_classify_general_band_layouts_search_mode(dev, oracle_lib):
    """The general (R = 26-30, two groups per warp) band layouts in SEARCH mode with several
    items per group (next-item setup, live best-so-far skip, near-tie log): windows 192-255 at
    L = 300 through classify against the exhaustive oracle."""
    ds = datagen.make_dataset(3, n_train=600)
    X, lab = ds.train, ds.train_labels
    Q, Tr, trl = X[:48], X[48:], lab[48:]
    for w in (192, 210, 225, 255):
        idx, lb_, dist, st = _classify(dev, Tr, trl, Q, w, 5, stats=True)
        assert st["dtw_calls"] > 4 * 148  # more items than groups: groups move on
        _check_nn(oracle_lib, Tr, trl, Q, w, idx, lb_, dist)
