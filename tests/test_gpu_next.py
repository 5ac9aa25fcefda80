"""GPU parity for SURVEY.md §8(f)'s next rows through the C ABI, against the fp64 oracle:
symmetric LB_Enhanced (NEXT-2), the tightness reduction (NEXT-3), LB_Improved (O(L) projection
envelope), LB_New and LB_Enhanced with the LB_Improved bridge (NEXT-4), and classify with every
alternative S2 bound including none (NEXT-1).  Bounds within relative 1e-5 (fp32 storage and accumulation, as for S2); NN indices
and labels bit-exact; tightness means within 1e-5 relative, pair counts exact."""
import numpy as np
import pytest

import datagen

from test_gpu_parity import REL, T, _check_nn, assert_rel, dev  # noqa: F401

pytestmark = pytest.mark.gpu


def _sets(seed, nq, nt, L, kinds=("walk", "int")):
    rng = np.random.default_rng(seed)
    Q = np.concatenate([datagen.random_series(rng, nq // len(kinds), L, k) for k in kinds])
    Tn = np.concatenate([datagen.random_series(rng, nt // len(kinds), L, k) for k in kinds])
    return Q, Tn


SHAPES = [(2, 0), (3, 1), (5, 4), (17, 3), (64, 0), (64, 63), (128, 13), (256, 26), (300, 30)]
# LB_Improved's van Herk scans: chunks of 128 elements per warp, blocks of 2w+1 aligned at -w;
# lengths around the chunk size, windows whose blocks straddle chunks and the row end
IMP_SHAPES = SHAPES + [(127, 5), (128, 64), (129, 1), (200, 199), (257, 12), (384, 100),
                       (512, 103), (1000, 333), (2048, 409), (2048, 2047),
                       (5000, 700)]  # > 4608: one pair per warp (the two-pair rows do not fit)


@pytest.mark.parametrize("L,w", SHAPES)
def test_lb_new_parity(dev, oracle_lib, L, w):
    from paper_1808_09617_b200 import nndtw
    Q, Tn = _sets(L * 7 + w, 12, 34, L)
    lb = nndtw.lb_new(T(Q, dev), T(Tn, dev), w).cpu().numpy()
    assert_rel(lb, oracle_lib.bound_matrix("new", Q, Tn, w), what="LB_New")


@pytest.mark.parametrize("L,w", IMP_SHAPES)
def test_lb_improved_parity(dev, oracle_lib, L, w):
    from paper_1808_09617_b200 import nndtw
    nq, nt = (12, 34) if L <= 512 else ((4, 10) if L <= 2048 else (3, 5))
    Q, Tn = _sets(L * 5 + w, nq, nt, L)
    lb = nndtw.lb_improved(T(Q, dev), T(Tn, dev), w).cpu().numpy()
    assert_rel(lb, oracle_lib.bound_matrix("improved", Q, Tn, w), what="LB_Improved")


@pytest.mark.parametrize("L,w", IMP_SHAPES)
@pytest.mark.parametrize("V", [1, 5])
def test_lb_enhanced_improved_parity(dev, oracle_lib, L, w, V):
    from paper_1808_09617_b200 import nndtw
    nq, nt = (12, 34) if L <= 512 else ((4, 10) if L <= 2048 else (3, 5))
    Q, Tn = _sets(L * 3 + w + V, nq, nt, L)
    lb = nndtw.lb_enhanced_improved(T(Q, dev), T(Tn, dev), w, V).cpu().numpy()
    assert_rel(lb, oracle_lib.bound_matrix("enhanced_improved", Q, Tn, w, V),
               what="LB_Enhanced with the LB_Improved bridge")


@pytest.mark.parametrize("bound", ["improved", "new", "enhanced_improved", "none"])
def test_classify_alternative_bounds_same_answer(dev, oracle_lib, bound):
    """Every S2 bound (and none) gives the exact 1-NN: configs 0/1 and an integer tie grid."""
    from paper_1808_09617_b200 import nndtw
    cases = [(0, 100, 10), (1, 80, 20), (1, 50, 1)]
    for cfg, nq, p in cases:
        ds = datagen.make_dataset(cfg)
        w = ds.cfg.windows()[0] if cfg == 0 else datagen.window_from_percent(p, 256)
        model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5, bound=bound)
        pred = nndtw.classify(model, T(ds.test[:nq], dev), stats=True, level_stats=True)
        _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test[:nq], w,
                  pred.idx.cpu().numpy(), pred.label.cpu().numpy(), pred.dist.cpu().numpy())
        st = pred.stats
        pruned = st["pruned_kim"] + st["pruned_bands"] + st["pruned_keogh"]
        assert pruned + st["survivors"] + nq == st["lb_pairs"], (bound, st)
        if bound == "none":
            assert pruned == 0 and st["survivors"] == st["lb_pairs"] - nq
    rng = np.random.default_rng(91)
    Tr = datagen.random_series(rng, 70, 29, "int")
    Tr = np.concatenate([Tr, Tr[:20]])
    Q = datagen.random_series(rng, 30, 29, "int")
    lab = np.arange(Tr.shape[0], dtype=np.int32) % 5
    model = nndtw.Model(T(Tr, dev), T(lab, dev), 3, 2, bound=bound)
    pred = nndtw.classify(model, T(Q, dev))
    _check_nn(oracle_lib, Tr, lab, Q, 3, pred.idx.cpu().numpy(), pred.label.cpu().numpy(),
              pred.dist.cpu().numpy(), V=2)


@pytest.mark.parametrize("bound", ["improved", "enhanced_improved", "none"])
def test_loocv_style_self_exclusion_alternative_bounds(dev, oracle_lib, bound):
    """classify with self_offset (the leave-one-out self pair) under an alternative bound: the
    held-out series is never its own neighbour."""
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(3, n_train=150)
    X, lab = ds.train, ds.train_labels
    w = 15
    model = nndtw.Model(T(X, dev), T(lab, dev), w, 5, bound=bound)
    key, _, _ = nndtw.classify_keys(model, T(X, dev), exact=True, self_offset=0)
    idx, _, _ = nndtw.finalize(key, model.labels)
    _, rnn = oracle_lib.loocv(X, lab, [w], V=5)
    assert np.array_equal(idx.cpu().numpy(), rnn[0])


@pytest.mark.parametrize("L,w,V", [(2, 1, 1), (16, 3, 2), (64, 0, 5), (128, 13, 5),
                                   (256, 255, 8), (300, 30, 40), (512, 103, 5)])
def test_lb_symmetric_parity(dev, oracle_lib, L, w, V):
    from paper_1808_09617_b200 import nndtw
    Q, Tn = _sets(L + 3 * w + V, 10, 140, L)
    sym = nndtw.lb_enhanced_symmetric(T(Q, dev), T(Tn, dev), w, V).cpu().numpy()
    assert_rel(sym, oracle_lib.bound_matrix("sym", Q, Tn, w, V), what="symmetric LB_Enhanced")
    # with Kim the value is max(Kim, symmetric); Keogh variant: max of the two directions
    symk = nndtw.lb_enhanced_symmetric(T(Q, dev), T(Tn, dev), w, V, with_kim=True).cpu().numpy()
    kim = np.array([[oracle_lib.lb_kim_sum(a, b) for b in Tn] for a in Q])
    assert_rel(symk, np.maximum(kim, oracle_lib.bound_matrix("sym", Q, Tn, w, V)),
               what="max(Kim, symmetric)")
    keo = nndtw.lb_enhanced_symmetric(T(Q, dev), T(Tn, dev), w, V, keogh=True).cpu().numpy()
    UQ, LQ = oracle_lib.envelopes(Q, w)
    UT, LT = oracle_lib.envelopes(Tn, w)
    ref = np.array([[max(oracle_lib.lb_keogh(a, UT[j], LT[j]), oracle_lib.lb_keogh(b, UQ[i], LQ[i]))
                     for j, b in enumerate(Tn)] for i, a in enumerate(Q)])
    assert_rel(keo, ref, what="symmetric LB_Keogh")


def test_classify_symmetric_same_answer(dev, oracle_lib):
    from paper_1808_09617_b200 import nndtw
    for cfg, nq, p in ((0, 100, 10), (1, 60, 20), (1, 40, 1)):
        ds = datagen.make_dataset(cfg)
        w = ds.cfg.windows()[0] if cfg == 0 else datagen.window_from_percent(p, 256)
        for bound in ("enhanced", "keogh"):
            model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5, bound=bound,
                                symmetric=True)
            pred = nndtw.classify(model, T(ds.test[:nq], dev), stats=True)
            _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test[:nq], w,
                      pred.idx.cpu().numpy(), pred.label.cpu().numpy(),
                      pred.dist.cpu().numpy())


def test_classify_symmetric_ties(dev, oracle_lib):
    """Integer grids with duplicates: many exact ties, lowest index must win."""
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(77)
    Tr = datagen.random_series(rng, 90, 33, "int")
    Tr = np.concatenate([Tr, Tr[:30]])
    Q = datagen.random_series(rng, 40, 33, "int")
    lab = np.arange(Tr.shape[0], dtype=np.int32) % 7
    model = nndtw.Model(T(Tr, dev), T(lab, dev), 4, 3, symmetric=True)
    pred = nndtw.classify(model, T(Q, dev))
    _check_nn(oracle_lib, Tr, lab, Q, 4, pred.idx.cpu().numpy(), pred.label.cpu().numpy(),
              pred.dist.cpu().numpy(), V=3)


@pytest.mark.parametrize("L,w", [(64, 6), (256, 26)])
def test_tightness_parity(dev, oracle_lib, L, w):
    """Mean sqrt(LB/DTW) over all pairs from the GPU bounds + GPU DTW equals the oracle's
    from its own bounds and exhaustive DTW; every ratio <= 1 (admissibility) up to rounding."""
    import torch
    from paper_1808_09617_b200 import nndtw
    Q, Tn = _sets(L + w, 16, 40, L, kinds=("walk",))
    q, t = T(Q, dev), T(Tn, dev)
    nq, nt = Q.shape[0], Tn.shape[0]
    ia = torch.arange(nq, device=dev, dtype=torch.int32).repeat_interleave(nt)
    ib = torch.arange(nt, device=dev, dtype=torch.int32).repeat(nq)
    d = nndtw.dtw_batch(q, t, w, ia, ib)
    dref = np.array([[oracle_lib.dtw(a, b, w) for b in Tn] for a in Q])
    assert_rel(d.cpu().numpy(), dref.ravel(), what="all-pairs DTW")
    U, Lo, kim = nndtw.envelopes(t, w)
    gpu_bounds = {
        "keogh": nndtw.lb_enhanced(q, t, U, Lo, w, 5, keogh=True),
        "enhanced": nndtw.lb_enhanced(q, t, U, Lo, w, 5),
        "improved": nndtw.lb_improved(q, t, w),
        "enhanced_improved": nndtw.lb_enhanced_improved(q, t, w, 5),
        "new": nndtw.lb_new(q, t, w),
        "sym": nndtw.lb_enhanced_symmetric(q, t, w, 5),
    }
    for kind, lb in gpu_bounds.items():
        mean, cnt, mx = nndtw.tightness(lb, d)
        ref_mean, ref_cnt = oracle_lib.tightness(oracle_lib.bound_matrix(kind, Q, Tn, w), dref)
        assert cnt == ref_cnt == nq * nt
        assert abs(mean - ref_mean) <= 1e-5 * ref_mean, (kind, mean, ref_mean)
        assert mx <= 1.0 + 1e-5, (kind, mx)
