"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle, element by element on
the same seeded inputs.  Tolerances: envelopes and NN indices/labels bit-exact; distances and
bounds within relative 1e-5 (north_star; fp32 storage and accumulation)."""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu

REL = 1e-5


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1808_09617_b200 import build, nndtw
    build.build()
    nndtw.load()
    assert nndtw.load().nndtw_check_device() == 0, "not an sm_100 device"
    return torch.device("cuda:0")


def T(x, dev):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), device=dev)


def assert_rel(gpu, ref, rel=REL, what=""):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(gpu - ref)
    tol = rel * np.abs(ref) + 1e-30
    bad = np.where(err > tol)[0] if gpu.ndim == 1 else np.argwhere(err > tol)
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}, " \
        f"max rel {np.max(err / np.maximum(np.abs(ref), 1e-30)):.3g}"


# ---------------------------------------------------------------- S1 envelopes
@pytest.mark.parametrize("L", [2, 3, 4, 7, 31, 128, 129, 255, 256, 300, 512, 513, 1000, 2048,
                               4100, 8192])
def test_envelopes_bit_exact(dev, oracle_lib, L):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L)
    X = np.concatenate([datagen.random_series(rng, 5, L, k) for k in ("walk", "int", "const")])
    for w in sorted({0, 1, 2, 3, L // 10, L // 5, L // 2, L - 2, L - 1, L, 5 * L}):
        if w < 0:
            continue
        U, Lo, kim = nndtw.envelopes(T(X, dev), w)
        eu, el = oracle_lib.envelopes(X, w)
        assert np.array_equal(U.cpu().numpy(), eu), (L, w)
        assert np.array_equal(Lo.cpu().numpy(), el), (L, w)
    k = kim.cpu().numpy()
    assert np.array_equal(k[:, 2], np.argmin(X, axis=1))
    assert np.array_equal(k[:, 3], np.argmax(X, axis=1))
    assert np.array_equal(k[:, 0].view(np.float32), X.min(axis=1))


@pytest.mark.parametrize("L", [257, 300, 512, 513, 1000, 2048])
def test_envelopes_direct_residues(dev, oracle_lib, L):
    """The direct (w >= 16) envelope kernel is instantiated per R = w mod 16: every residue, the
    smallest q, windows near L, and the Kim features of every call."""
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L + 1)
    X = np.concatenate([datagen.random_series(rng, 7, L, k) for k in ("walk", "int")])
    ws = list(range(16, 48)) + [103, L // 3, L // 2 + 5, L - 17, L - 2]
    for w in sorted(set(ws)):
        U, Lo, kim = nndtw.envelopes(T(X, dev), w)
        eu, el = oracle_lib.envelopes(X, w)
        assert np.array_equal(U.cpu().numpy(), eu), (L, w)
        assert np.array_equal(Lo.cpu().numpy(), el), (L, w)
        k = kim.cpu().numpy()
        assert np.array_equal(k[:, 2], np.argmin(X, axis=1)), (L, w)
        assert np.array_equal(k[:, 3], np.argmax(X, axis=1)), (L, w)
        assert np.array_equal(k[:, 0].view(np.float32), X.min(axis=1)), (L, w)
        assert np.array_equal(k[:, 1].view(np.float32), X.max(axis=1)), (L, w)


def test_envelopes_many_sets(dev, oracle_lib):
    """More series than resident blocks: the persistent kernels loop over series sets."""
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(5)
    L = 512
    X = datagen.random_series(rng, 6001, L, "walk")
    for w in (5, 51, 103):
        U, Lo, kim = nndtw.envelopes(T(X, dev), w)
        eu, el = oracle_lib.envelopes(X, w)
        assert np.array_equal(U.cpu().numpy(), eu), w
        assert np.array_equal(Lo.cpu().numpy(), el), w
        assert np.array_equal(kim.cpu().numpy()[:, 3], np.argmax(X, axis=1)), w


# ---------------------------------------------------------------- S2 bounds
@pytest.mark.parametrize("L,w,V", [(2, 0, 1), (3, 1, 2), (16, 3, 5), (64, 0, 5), (100, 7, 3),
                                   (128, 13, 5), (256, 255, 8), (300, 30, 40), (512, 103, 5),
                                   (200, 199, 100)])
def test_lb_enhanced_parity(dev, oracle_lib, L, w, V):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L * 7 + w)
    Q = datagen.random_series(rng, 70, L, "walk")
    Tn = datagen.random_series(rng, 150, L, "walk")
    Tn[5] = Q[3]
    qt, tt = T(Q, dev), T(Tn, dev)
    U, Lo, kim = nndtw.envelopes(tt, w)
    lb = nndtw.lb_enhanced(qt, tt, U, Lo, w, V).cpu().numpy()
    lbk = nndtw.lb_enhanced(qt, tt, U, Lo, w, V, with_kim=True, tkim=kim).cpu().numpy()
    eu, el = oracle_lib.envelopes(Tn, w)
    for i in range(0, 70, 3):
        for j in range(150):
            ref, _ = oracle_lib.lb_enhanced(Q[i], Tn[j], eu[j], el[j], w, V)
            refk = max(ref, oracle_lib.lb_kim_sum(Q[i], Tn[j]))
            assert abs(lb[i, j] - ref) <= REL * ref + 1e-30, (i, j, lb[i, j], ref)
            assert abs(lbk[i, j] - refk) <= REL * refk + 1e-30, (i, j, lbk[i, j], refk)


@pytest.mark.parametrize("L,w,V", [(2, 1, 5), (9, 2, 3), (64, 6, 5), (300, 30, 16),
                                   (512, 103, 5), (257, 0, 4), (128, 127, 40)])
def test_lb_enhanced_partial_parity(dev, oracle_lib, L, w, V):
    """NNDTW_LB_PARTIAL (stage A of the two-stage S2): Algorithm 1 up to its line-12 test.  The
    oracle's value is its own Algorithm 1 with an envelope of (+inf, -inf) -- every LB_Keogh
    bridge term (lines 13-15) is then zero -- and it must not exceed the full bound."""
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L * 11 + w)
    Q = datagen.random_series(rng, 40, L, "walk")
    Tn = datagen.random_series(rng, 90, L, "walk")
    Tn[4] = Q[2]
    qt, tt = T(Q, dev), T(Tn, dev)
    U, Lo, kim = nndtw.envelopes(tt, w)
    part = nndtw.lb_enhanced(qt, tt, U, Lo, w, V, partial=True).cpu().numpy()
    partk = nndtw.lb_enhanced(qt, tt, U, Lo, w, V, with_kim=True, tkim=kim,
                              partial=True).cpu().numpy()
    full = nndtw.lb_enhanced(qt, tt, U, Lo, w, V).cpu().numpy()
    inf_u = np.full(L, np.inf, dtype=np.float32)
    for i in range(0, 40, 3):
        for j in range(90):
            ref, _ = oracle_lib.lb_enhanced(Q[i], Tn[j], inf_u, -inf_u, w, V)
            refk = max(ref, oracle_lib.lb_kim_sum(Q[i], Tn[j]))
            assert abs(part[i, j] - ref) <= REL * ref + 1e-30, (i, j, part[i, j], ref)
            assert abs(partk[i, j] - refk) <= REL * refk + 1e-30, (i, j, partk[i, j], refk)
    assert np.all(part <= full * (1 + REL) + 1e-30)


# ---------------------------------------------------------------- S4 DTW
@pytest.mark.parametrize("L", [2, 3, 5, 17, 64, 128, 256, 300, 512])
def test_dtw_batch_parity(dev, oracle_lib, L):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(100 + L)
    A = datagen.random_series(rng, 24, L, "walk")
    B = datagen.random_series(rng, 24, L, "walk")
    B[0] = A[0]
    for w in sorted({0, 1, 2, 3, L // 8, L // 4, L // 2, L - 1, L + 3}):
        out = nndtw.dtw_batch(T(A, dev), T(B, dev), w).cpu().numpy()
        ref = np.array([oracle_lib.dtw(A[p], B[p], w) for p in range(24)])
        assert_rel(out, ref, what=f"L={L} w={w}")


def test_dtw_batch_indexed_and_abandon(dev, oracle_lib):
    import torch
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(7)
    L, w = 200, 20
    A = datagen.random_series(rng, 10, L, "walk")
    B = datagen.random_series(rng, 30, L, "walk")
    ia = rng.integers(0, 10, size=300).astype(np.int32)
    ib = rng.integers(0, 30, size=300).astype(np.int32)
    ref = np.array([oracle_lib.dtw(A[i], B[j], w) for i, j in zip(ia, ib)])
    cut = (ref * rng.uniform(0.3, 1.6, size=300)).astype(np.float32)
    out = nndtw.dtw_batch(T(A, dev), T(B, dev), w, ia=T(ia, dev), ib=T(ib, dev),
                          cutoff=T(cut, dev)).cpu().numpy()
    aband = np.isinf(out)
    assert np.all(ref[aband] > cut[aband])          # abandoned => exact value > cutoff
    assert_rel(out[~aband], ref[~aband], what="non-abandoned")
    assert aband.sum() > 10                          # abandoning is effective
    full = nndtw.dtw_batch(T(A, dev), T(B, dev), w, ia=T(ia, dev), ib=T(ib, dev)).cpu().numpy()
    assert_rel(full, ref, what="no cutoff")


# ---------------------------------------------------------------- S2-S7 classify
def _classify(dev, Tr, trl, Q, w, V, stats=False):
    from paper_1808_09617_b200 import nndtw
    model = nndtw.Model(T(Tr, dev), T(trl, dev), w, V)
    pred = nndtw.classify(model, T(Q, dev), stats=stats)
    return (pred.idx.cpu().numpy(), pred.label.cpu().numpy(), pred.dist.cpu().numpy(),
            pred.stats)


def _check_nn(oracle_lib, Tr, trl, Q, w, idx, lab, dist, mode="exhaustive", V=5):
    ridx, rdist = oracle_lib.nn(Q, Tr, w, V=V, mode=mode)
    assert np.array_equal(idx, ridx), np.nonzero(idx != ridx)[0][:10]
    assert np.array_equal(lab, trl[ridx])
    assert_rel(dist, rdist, what="nn distance")


def test_classify_config0(dev, oracle_lib):
    ds = datagen.make_dataset(0)
    w = ds.cfg.windows()[0]
    idx, lab, dist, st = _classify(dev, ds.train, ds.train_labels, ds.test, w, 5, stats=True)
    _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test, w, idx, lab, dist)
    assert st["lb_pairs"] == 100 * 100 and st["dtw_calls"] < 100 * 100


@pytest.mark.parametrize("p", [1, 10, 20, 50, 100])
def test_classify_config1_grid(dev, oracle_lib, p):
    """BJ:configs[1] at full N=1000 train, a 120-query sample, every V of the grid."""
    ds = datagen.make_dataset(1)
    w = datagen.window_from_percent(p, 256)
    Q = ds.test[:120]
    ridx, rdist = oracle_lib.nn(Q, ds.train, w, mode="pruned")
    for V in ds.cfg.Vs:
        idx, lab, dist, _ = _classify(dev, ds.train, ds.train_labels, Q, w, V)
        assert np.array_equal(idx, ridx), (V, np.nonzero(idx != ridx)[0][:10])
        assert_rel(dist, rdist, what=f"p={p} V={V}")


@pytest.mark.parametrize("kind,L,w,V", [("int", 8, 2, 3), ("int", 16, 0, 5), ("int", 33, 32, 4),
                                        ("walk", 2, 0, 1), ("walk", 3, 1, 5), ("const", 12, 3, 2),
                                        ("walk", 130, 129, 70), ("int", 64, 5, 1),
                                        ("int", 300, 40, 5), ("walk", 600, 599, 5),
                                        ("walk", 1024, 200, 5)])
def test_classify_ties_and_edges(dev, oracle_lib, kind, L, w, V):
    """Exact ties (integer grids, duplicates, constants): the lowest train index must win.
    (L > 256: the fp64 re-rank of the near-tie sets runs one warp per 256-row strip,
    k_refine_cta; the full window at L = 600 also goes through the row-strip kernel.)"""
    rng = np.random.default_rng(L * 31 + w)
    Tr = datagen.random_series(rng, 257, L, kind)
    Tr[200:210] = Tr[17]          # duplicates after the original
    Tr[3] = Tr[250]               # duplicate before
    Q = datagen.random_series(rng, 61, L, kind)
    Q[0] = Tr[17]
    trl = rng.integers(0, 4, size=257).astype(np.int32)
    idx, lab, dist, _ = _classify(dev, Tr, trl, Q, w, V)
    _check_nn(oracle_lib, Tr, trl, Q, w, idx, lab, dist)


def test_classify_single_pair(dev, oracle_lib):
    rng = np.random.default_rng(3)
    Tr = datagen.random_series(rng, 1, 50, "walk")
    Q = datagen.random_series(rng, 1, 50, "walk")
    idx, lab, dist, _ = _classify(dev, Tr, np.array([7], np.int32), Q, 5, 5)
    assert idx[0] == 0 and lab[0] == 7
    assert_rel(dist, [oracle_lib.dtw(Q[0], Tr[0], 5)])


@pytest.mark.slow
def test_classify_config2_full_sampled(dev, oracle_lib):
    """BJ:configs[2] at full size (1e4 queries x 1e5 train, L=512, w=103, V=5) in the bench's
    launch configuration; a seeded sample of queries is checked against the oracle's pruned
    search (itself pinned to exhaustive search in test_oracle_pins)."""
    ds = datagen.make_dataset(2)
    w = ds.cfg.windows()[0]
    idx, lab, dist, st = _classify(dev, ds.train, ds.train_labels, ds.test, w, 5, stats=True)
    rng = np.random.default_rng(2)
    sample = np.sort(rng.choice(ds.test.shape[0], size=16, replace=False))
    ridx, rdist = oracle_lib.nn(ds.test[sample], ds.train, w, V=5, mode="pruned")
    assert np.array_equal(idx[sample], ridx)
    assert_rel(dist[sample], rdist, what="config 2 sample")
    acc = np.mean(lab == ds.test_labels)
    assert acc > 0.9
    assert st["dtw_calls"] < 0.2 * st["lb_pairs"]


# ---------------------------------------------------------------- S8 LOOCV
def test_loocv_reduced(dev, oracle_lib):
    import torch
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(3, n_train=240)
    X, lab = ds.train, ds.train_labels
    windows = [datagen.window_from_percent(p, 300) for p in (0, 1, 2, 5, 10, 30, 100)]
    err, nn, _ = nndtw.loocv_window(T(X, dev), T(lab, dev), windows, v=5, with_nn=True)
    rerr, rnn = oracle_lib.loocv(X, lab, windows, V=5, mode="pruned")
    assert np.array_equal(nn.cpu().numpy(), rnn.astype(np.int32))
    assert np.array_equal(err.cpu().numpy(), rerr)
    # a query shard [60, 170) gives the same rows
    err2, nn2, _ = nndtw.loocv_window(T(X, dev), T(lab, dev), windows, v=5, q_begin=60,
                                      q_end=170, with_nn=True)
    assert np.array_equal(nn2.cpu().numpy(), rnn[:, 60:170].astype(np.int32))


# ---------------------------------------------------------------- S4 long windows (strip kernel)
# rows per lane RR (strip_rows_per_lane) and sub-blocks KS: 1024/2048/3001 -> RR 32, KS 4;
# 700/1100 -> 12, 4; 513/600 -> 10, 2; 1792/256 -> 8, 4; each with and without the band mask
@pytest.mark.parametrize("L,ws", [(1024, (1023, 600, 515)), (2048, (2047, 1500)),
                                  (700, (699, 520)), (1100, (1099,)), (513, (512,)),
                                  (600, (599, 520)), (1792, (1791, 600)), (256, (255,)),
                                  (3001, (3000, 2000)),
                                  # band kernel, general layouts wider than R = 24 (two groups
                                  # per warp from 2w+2 > 384, one group up to 2w+2 = 960)
                                  (300, (192, 210, 225, 255)), (1024, (200, 400)),
                                  (2048, (409,))])
def test_dtw_batch_long_windows(dev, oracle_lib, L, ws):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L)
    A = datagen.random_series(rng, 6, L, "walk")
    B = datagen.random_series(rng, 6, L, "walk")
    B[1] = A[1]
    for w in ws:
        out = nndtw.dtw_batch(T(A, dev), T(B, dev), w).cpu().numpy()
        ref = np.array([oracle_lib.dtw(A[p], B[p], w) for p in range(6)])
        assert_rel(out, ref, what=f"L={L} w={w}")
        cut = (ref * np.array([0.3, 2.0, 0.9, 1.1, 0.5, 1.5])).astype(np.float32)
        out2 = nndtw.dtw_batch(T(A, dev), T(B, dev), w, cutoff=T(cut, dev)).cpu().numpy()
        ab = np.isinf(out2)
        assert np.all(ref[ab] > cut[ab])
        assert_rel(out2[~ab], ref[~ab], what=f"L={L} w={w} cutoff")


def test_classify_long_window_small(dev, oracle_lib):
    ds = datagen.make_dataset(4, n_train=300, n_test=12)
    w = ds.cfg.windows()[0]
    idx, lab, dist, st = _classify(dev, ds.train, ds.train_labels, ds.test, w, 8, stats=True)
    _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test, w, idx, lab, dist)


@pytest.mark.slow
def test_classify_config4_full_sampled(dev, oracle_lib):
    """BJ:configs[4] at full size (1e3 queries x 1e4 train, L=2048, w=L-1, V=8); a seeded
    sample of queries checked against the oracle's pruned search."""
    ds = datagen.make_dataset(4)
    w = ds.cfg.windows()[0]
    idx, lab, dist, st = _classify(dev, ds.train, ds.train_labels, ds.test, w, 8, stats=True)
    rng = np.random.default_rng(4)
    sample = np.sort(rng.choice(ds.test.shape[0], size=6, replace=False))
    ridx, rdist = oracle_lib.nn(ds.test[sample], ds.train, w, V=8, mode="pruned")
    assert np.array_equal(idx[sample], ridx)
    assert_rel(dist[sample], rdist, what="config 4 sample")


@pytest.mark.slow
def test_loocv_config3_full_sampled(dev, oracle_lib):
    """BJ:configs[3] at full size (2000 series, all 101 windows): per-window NN ids of a seeded
    sample of held-out series are checked against the oracle (exhaustive over j != i)."""
    import torch
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(3)
    X, lab = ds.train, ds.train_labels
    wins = ds.cfg.windows()
    err, nn, _ = nndtw.loocv_window(T(X, dev), T(lab, dev), wins, v=5, with_nn=True)
    nn = nn.cpu().numpy()
    err = err.cpu().numpy()
    # error counts are consistent with the reported neighbours
    for p in range(len(wins)):
        assert err[p] == int(np.sum(lab[nn[p]] != lab))
    rng = np.random.default_rng(3)
    sample = rng.choice(X.shape[0], size=4, replace=False)
    widx = [0, 1, 7, 20, 50, 100]
    for i in sample:
        rerr, rnn = oracle_lib.loocv(X, lab, [wins[p] for p in widx], V=5, q_begin=int(i),
                                     q_end=int(i) + 1, mode="pruned")
        assert np.array_equal(nn[widx, i], rnn[:, 0].astype(np.int32)), (i, nn[widx, i], rnn[:, 0])


# ---------------------------------------------------------------- S6 shard protocol (1 GPU)
@pytest.mark.parametrize("nshards", [2, 3])
@pytest.mark.parametrize("two_phase", [False, True, "split"])
@pytest.mark.parametrize("data", ["int", "config1"])
def test_shard_protocol_through_abi(dev, oracle_lib, nshards, two_phase, data):
    """The sharded path of dist.py through the real C ABI, shards run one after another on one
    GPU and combined with torch.minimum (= the int64 MIN all-reduce): refine and resolve must
    give the exact global 1-NN, including exact ties split across shards.  two_phase: the seed
    keys are MIN-combined first and every shard searches from the global seed; "split": the
    search in two halves (PHASE_SEARCH_A / _B) with another MIN between them."""
    import torch
    from paper_1808_09617_b200 import nndtw
    from paper_1808_09617_b200.dist import shard_range
    rng = np.random.default_rng(nshards)
    if data == "int":
        L, w, V, N = 64, 6, 5, 300
        Tr = datagen.random_series(rng, N, L, "int")
        Tr[250] = Tr[20]      # duplicates in different shards
        Tr[299] = Tr[120]
        Q = datagen.random_series(rng, 40, L, "int")
        Q[0] = Tr[20]
        Q[1] = Tr[120]
        labels = rng.integers(0, 5, size=N).astype(np.int32)
    else:  # config-1 shaped (pruning and abandoning at work)
        ds = datagen.make_dataset(1, n_train=1000, n_test=60)
        Tr, Q, labels = ds.train, ds.test, ds.train_labels
        N, L, w, V = 1000, 256, 26, 5
    q = T(Q, dev)
    models = []
    for r in range(nshards):
        lo, hi = shard_range(N, r, nshards)
        models.append(nndtw.Model(T(Tr[lo:hi], dev), T(labels[lo:hi], dev), w, V, index_base=lo))
    if two_phase:
        seeds = [nndtw.classify_keys(m, q, exact=False, phase="seed") for m in models]
        gseed = seeds[0][0].clone()
        for k, _, _ in seeds[1:]:
            gseed = torch.minimum(gseed, k)
        if two_phase == "split":
            mids = [nndtw.classify_keys(m, q, exact=False, phase="search_a", key=gseed.clone(),
                                        ws=ws) for m, (_, ws, _) in zip(models, seeds)]
            gmid = mids[0][0].clone()
            for k, _, _ in mids[1:]:
                gmid = torch.minimum(gmid, k)
            outs = [nndtw.classify_keys(m, q, exact=False, phase="search_b", key=gmid.clone(),
                                        ws=ws) for m, (_, ws, _) in zip(models, seeds)]
        else:
            outs = [nndtw.classify_keys(m, q, exact=False, phase="search", key=gseed.clone(),
                                        ws=ws) for m, (_, ws, _) in zip(models, seeds)]
    else:
        outs = [nndtw.classify_keys(m, q, exact=False) for m in models]
    gkey = outs[0][0].clone()
    for k, _, _ in outs[1:]:
        gkey = torch.minimum(gkey, k)
    f64 = [nndtw.classify_refine(m, q, ws, gkey) for m, (_, ws, _) in zip(models, outs)]
    gf64 = f64[0].clone()
    for x in f64[1:]:
        gf64 = torch.minimum(gf64, x)
    res = [nndtw.classify_resolve(m, q, ws, gkey, gf64) for m, (_, ws, _) in zip(models, outs)]
    g = res[0].clone()
    for x in res[1:]:
        g = torch.minimum(g, x)
    idx, lab, dist = nndtw.finalize(g, T(labels, dev), key_format=1)
    _check_nn(oracle_lib, Tr, labels, Q, w, idx.cpu().numpy(), lab.cpu().numpy(),
              dist.cpu().numpy(), V=V)


# ---------------------------------------------------------------- NEXT-1: LB_Keogh baseline
@pytest.mark.parametrize("L,w", [(16, 3), (128, 13), (300, 299), (512, 103)])
def test_lb_keogh_parity(dev, oracle_lib, L, w):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(L + w)
    Q = datagen.random_series(rng, 40, L, "walk")
    Tn = datagen.random_series(rng, 130, L, "walk")
    U, Lo, kim = nndtw.envelopes(T(Tn, dev), w)
    lb = nndtw.lb_enhanced(T(Q, dev), T(Tn, dev), U, Lo, w, 5, keogh=True).cpu().numpy()
    eu, el = oracle_lib.envelopes(Tn, w)
    for i in range(0, 40, 3):
        for j in range(130):
            ref = oracle_lib.lb_keogh(Q[i], eu[j], el[j])
            assert abs(lb[i, j] - ref) <= REL * ref + 1e-30, (i, j, lb[i, j], ref)


def test_classify_keogh_bound_same_answer(dev, oracle_lib):
    from paper_1808_09617_b200 import nndtw
    for cfg, nq in ((0, 100), (1, 60)):
        ds = datagen.make_dataset(cfg)
        w = ds.cfg.windows()[0] if cfg == 0 else datagen.window_from_percent(20, 256)
        model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5, bound="keogh")
        pred = nndtw.classify(model, T(ds.test[:nq], dev), stats=True)
        _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test[:nq], w,
                  pred.idx.cpu().numpy(), pred.label.cpu().numpy(), pred.dist.cpu().numpy())


def test_classify_tie_log_overflow(dev, oracle_lib, monkeypatch):
    """Force the near-tie log to overflow (capacity 8 entries): the affected queries fall back
    to re-ranking every surviving candidate in fp64 (k_refine_overflow), same exact answer."""
    from paper_1808_09617_b200 import nndtw
    monkeypatch.setenv("NNDTW_TIE_LOG_CAP", "8")
    rng = np.random.default_rng(5)
    Tr = datagen.random_series(rng, 60, 24, "int")
    Tr = np.concatenate([Tr, Tr, Tr[:20]])          # every candidate has exact duplicates
    Q = np.concatenate([Tr[:10], datagen.random_series(rng, 20, 24, "int")])
    lab = (np.arange(Tr.shape[0]) % 5).astype(np.int32)
    for w in (0, 3, 23):
        model = nndtw.Model(T(Tr, dev), T(lab, dev), w, 3)
        pred = nndtw.classify(model, T(Q, dev))
        _check_nn(oracle_lib, Tr, lab, Q, w, pred.idx.cpu().numpy(), pred.label.cpu().numpy(),
                  pred.dist.cpu().numpy(), V=3)


def test_loocv_sharded_world1_nccl(dev, oracle_lib):
    """dist.loocv_sharded through the C ABI and a real one-rank NCCL group (the N>1 launch path of
    S8 at N=1): counts and best window equal the oracle's."""
    import socket

    import torch
    import torch.distributed as dist
    from paper_1808_09617_b200.dist import best_window, loocv_sharded
    rng = np.random.default_rng(11)
    X = datagen.random_series(rng, 90, 40, "walk")
    lab = (np.arange(90) % 4).astype(np.int32)
    wins = [0, 2, 4, 8, 20, 39]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=dev)
    try:
        errors, best = loocv_sharded(T(X, dev), T(lab, dev), wins, v=5)
    finally:
        dist.destroy_process_group()
    ref, _ = oracle_lib.loocv(X, lab, wins, V=5)
    assert errors.cpu().tolist() == list(ref)
    assert best == best_window(ref, wins)
