"""Pins for the fp64 oracle against things other than itself (CPU only).

Each pin is chosen so that a plausible mistake in oracle/nndtw_oracle.c fails it:
* DTW: brute-force enumeration of every warping path -- bit-exact, because the
  DP's cell value equals the min over paths of the rounded left-fold path sums (rounded
  addition of non-negative numbers is monotone); closed form W=0 = squared ED.
* Envelopes: numpy sliding_window_view max/min over the clipped window of Eq. 3-4.
* LB_Enhanced: Eq. 7 evaluated literally from the band SETS of P:313-314 / P:355
  (readings C8, C9) in exact rational arithmetic -- a different formulation from
  Algorithm 1's loops; Theorem 2 admissibility against brute force; W=0 collapse; V=1 >=
  LB_Keogh.
* NN: exhaustive search vs a brute-force argmin; the pruned search (P:567-570 + Alg. 1) vs
  exhaustive (pruning is lossless, Thm 2).
* SPEC worked examples (tests/golden/spec_examples.jsonl, each line cites its source).
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.jsonl")


# ---------------- independent reference implementations (tests only) ----------------

def brute_dtw(a, b, w):
    """min over all warping paths (boundary, continuity, monotonicity: P:119-120) inside the
    band |i-j| <= w of the fp64 left-fold sum delta_k + s_{k-1}."""
    a = [float(x) for x in np.asarray(a, dtype=np.float32)]
    b = [float(x) for x in np.asarray(b, dtype=np.float32)]
    L = len(a)
    w = min(w, L - 1)
    best = float("inf")

    def delta(i, j):
        d = a[i] - b[j]
        return d * d

    def rec(i, j, s):
        nonlocal best
        if i == L - 1 and j == L - 1:
            best = min(best, s)
            return
        for di, dj in ((1, 0), (0, 1), (1, 1)):
            ni, nj = i + di, j + dj
            if ni < L and nj < L and abs(ni - nj) <= w:
                rec(ni, nj, delta(ni, nj) + s)

    rec(0, 0, delta(0, 0))
    return best


def left_set(i, w, L):
    """L_i^W of P:313-314 (1-based): {(x,i): max(1,i-W)<=x<=i} U {(i,y): max(1,i-W)<=y<i}."""
    lo = max(1, i - w)
    return [(x, i) for x in range(lo, i + 1)] + [(i, y) for y in range(lo, i)]


def right_set(i, w, L):
    """R_i^W, reading C9 (Alg. 1 lines 5, 9, 10): {(x,i): i<=x<=min(L,i+W)} U
    {(i,y): i<y<=min(L,i+W)}."""
    hi = min(L, i + w)
    return [(x, i) for x in range(i, hi + 1)] + [(i, y) for y in range(i + 1, hi + 1)]


def eq7_exact(a, b, w, V):
    """Eq. 7 summed in exact rationals from the band sets and Eq. 3-4 envelopes,
    with V read as n_bands = min(floor(L/2), V) (reading C10)."""
    a = [Fraction(float(x)) for x in np.asarray(a, dtype=np.float32)]
    b = [Fraction(float(x)) for x in np.asarray(b, dtype=np.float32)]
    L = len(a)
    w = min(w, L - 1)
    nb = min(L // 2, V)
    d = lambda x, y: (a[x - 1] - b[y - 1]) ** 2  # noqa: E731  (link (x,y) aligns A_x with B_y)
    tot = Fraction(0)
    for i in range(1, L + 1):
        if i <= nb:
            tot += min(d(x, y) for x, y in left_set(i, w, L))
        elif i > L - nb:
            tot += min(d(x, y) for x, y in right_set(i, w, L))
        else:
            win = b[max(1, i - w) - 1:min(L, i + w)]
            U, Lo = max(win), min(win)
            if a[i - 1] > U:
                tot += (a[i - 1] - U) ** 2
            elif a[i - 1] < Lo:
                tot += (a[i - 1] - Lo) ** 2
    return tot


def np_envelope(b, w):
    b = np.asarray(b, dtype=np.float32)
    L = b.size
    w = min(w, L - 1)
    pad_hi = np.concatenate([np.full(w, -np.inf, np.float32), b, np.full(w, -np.inf, np.float32)])
    pad_lo = np.concatenate([np.full(w, np.inf, np.float32), b, np.full(w, np.inf, np.float32)])
    sw = np.lib.stride_tricks.sliding_window_view
    return sw(pad_hi, 2 * w + 1).max(axis=1), sw(pad_lo, 2 * w + 1).min(axis=1)


def np_keogh(a, b, w):
    U, Lo = np_envelope(b, w)
    a = np.asarray(a, dtype=np.float32).astype(np.float64)
    above = np.where(a > U, (a - U) ** 2, 0.0)
    below = np.where(a < Lo, (a - Lo) ** 2, 0.0)
    return float(np.sum(above + below))


def rng_pairs(seed, n, Lmax, kinds=("walk", "normal", "int")):
    rng = np.random.default_rng(seed)
    out = []
    for t in range(n):
        L = int(rng.integers(2, Lmax + 1))
        kind = kinds[t % len(kinds)]
        x = datagen.random_series(rng, 2, L, kind)
        out.append((x[0], x[1]))
    return out


# ------------------------------------------------------------------------------------

def test_golden_spec_examples(oracle_lib):
    o = oracle_lib
    n = 0
    with open(GOLDEN) as f:
        for line in f:
            ex = json.loads(line)
            op = ex["op"]
            if op == "dtw":
                assert o.dtw(ex["a"], ex["b"], ex["w"]) == ex["expected"], ex["cite"]
            elif op == "sqed":
                assert o.sqed(ex["a"], ex["b"]) == ex["expected"], ex["cite"]
            elif op == "envelope":
                U, Lo = o.envelope(ex["b"], ex["w"])
                assert U.tolist() == ex["upper"] and Lo.tolist() == ex["lower"], ex["cite"]
            elif op == "kim":
                assert o.lb_kim_sum(ex["a"], ex["b"]) == ex["expected"], ex["cite"]
            elif op == "keogh":
                U, Lo = o.envelope(ex["b"], ex["w"])
                assert o.lb_keogh(ex["a"], U, Lo) == ex["expected"], ex["cite"]
            elif op == "band_left":
                # Alg. 1 with V=i, W=w accumulates the left band i; check via Eq. 7 sets
                a, b, i, w = ex["a"], ex["b"], ex["i"], ex["w"]
                m = min((a[x - 1] - b[y - 1]) ** 2 for x, y in left_set(i, w, len(a)))
                assert m == ex["expected"], ex["cite"]
            elif op == "lb_enhanced":
                U, Lo = o.envelope(ex["b"], ex["w"])
                v, ab = o.lb_enhanced(ex["a"], ex["b"], U, Lo, ex["w"], ex["V"])
                assert not ab and v == ex["expected"], ex["cite"]
            else:
                raise AssertionError(op)
            n += 1
    assert n >= 15


def test_dtw_equals_path_enumeration_bit_exact(oracle_lib):
    for a, b in rng_pairs(1, 260, 6):
        L = a.size
        for w in range(0, L + 1):
            assert oracle_lib.dtw(a, b, w) == brute_dtw(a, b, w), (a, b, w)


def test_dtw_L7_enumeration(oracle_lib):
    for a, b in rng_pairs(2, 12, 7):
        for w in (0, 1, 2, 6):
            assert oracle_lib.dtw(a, b, w) == brute_dtw(a, b, w)


def test_dtw_closed_forms_and_invariants(oracle_lib):
    rng = np.random.default_rng(3)
    for t in range(60):
        L = int(rng.integers(2, 40))
        a, b = datagen.random_series(rng, 2, L, ("walk", "normal", "int")[t % 3])
        # W = 0 is the squared Euclidean distance, summed left to right in fp64
        s = 0.0
        for x, y in zip(a.astype(np.float64), b.astype(np.float64)):
            s = (x - y) * (x - y) + s
        assert oracle_lib.dtw(a, b, 0) == s
        # symmetric; non-increasing in W; W >= L-1 is unconstrained
        prev = float("inf")
        for w in range(0, L + 2):
            d = oracle_lib.dtw(a, b, w)
            assert d == oracle_lib.dtw(b, a, w)
            assert d <= prev
            prev = d
        assert oracle_lib.dtw(a, b, L - 1) == oracle_lib.dtw(a, b, 10 * L)
        assert oracle_lib.dtw(a, a, int(rng.integers(0, L))) == 0.0


def test_dtw_abandon_sound(oracle_lib):
    rng = np.random.default_rng(4)
    for t in range(200):
        L = int(rng.integers(2, 30))
        a, b = datagen.random_series(rng, 2, L, "walk")
        w = int(rng.integers(0, L))
        d = oracle_lib.dtw(a, b, w)
        cut = d * float(rng.uniform(0.2, 1.5))
        v, ab, _ = oracle_lib.dtw_cut(a, b, w, cut)
        if ab:
            assert d > cut and v == float("inf")
        else:
            assert v == d
        v, ab, _ = oracle_lib.dtw_cut(a, b, w, d)  # cutoff == value never abandons
        assert not ab and v == d


def test_envelopes_vs_sliding_window(oracle_lib):
    rng = np.random.default_rng(5)
    for t in range(120):
        L = int(rng.integers(1, 80))
        b = datagen.random_series(rng, 1, L, ("walk", "int", "const")[t % 3])[0]
        for w in {0, 1, 2, L // 3, L - 1, L, 3 * L}:
            U, Lo = oracle_lib.envelope(b, w)
            eu, el = np_envelope(b, w)
            assert np.array_equal(U, eu) and np.array_equal(Lo, el)
            assert np.all(Lo <= b) and np.all(b <= U)


def test_keogh_vs_numpy(oracle_lib):
    for a, b in rng_pairs(6, 100, 50):
        for w in (0, 1, 3, a.size - 1):
            U, Lo = oracle_lib.envelope(b, w)
            assert oracle_lib.lb_keogh(a, U, Lo) == pytest.approx(np_keogh(a, b, w), rel=1e-12,
                                                                  abs=0)


def test_alg1_equals_eq7_literal_sets(oracle_lib):
    """Algorithm 1 == Eq. 7 evaluated from the band sets, exactly up to fp64
    rounding of the sums, over all W and V for L <= 9."""
    for a, b in rng_pairs(7, 70, 9):
        L = a.size
        for w in range(0, L + 1):
            U, Lo = oracle_lib.envelope(b, w)
            for V in range(1, L // 2 + 3):
                v, ab = oracle_lib.lb_enhanced(a, b, U, Lo, w, V)
                exact = eq7_exact(a, b, w, V)
                assert not ab
                assert abs(v - float(exact)) <= 1e-12 * max(1.0, float(exact)), (a, b, w, V)


def test_lb_admissible_and_reductions(oracle_lib):
    """Thm 2: LB_Enhanced <= DTW_W; Kim sum <= DTW; V=1 >= LB_Keogh;
    W=0 collapses LB_Enhanced to the squared ED; V >= L/2 gives bands only."""
    for t, (a, b) in enumerate(rng_pairs(8, 150, 7)):
        L = a.size
        for w in range(0, L):
            U, Lo = oracle_lib.envelope(b, w)
            d = brute_dtw(a, b, w)
            tol = 1e-12 * max(1.0, d)
            assert oracle_lib.lb_kim_sum(a, b) <= d + tol
            for V in range(1, L // 2 + 1):
                v, _ = oracle_lib.lb_enhanced(a, b, U, Lo, w, V)
                assert v <= d + tol, (a, b, w, V, v, d)
            v1, _ = oracle_lib.lb_enhanced(a, b, U, Lo, w, 1)
            assert v1 >= oracle_lib.lb_keogh(a, U, Lo) - tol
        U, Lo = oracle_lib.envelope(b, 0)
        for V in (1, 2, L):
            v, _ = oracle_lib.lb_enhanced(a, b, U, Lo, 0, V)
            assert v == pytest.approx(oracle_lib.sqed(a, b), rel=1e-12, abs=1e-300)


def test_kim_admissible_random(oracle_lib):
    rng = np.random.default_rng(9)
    for t in range(3000):
        L = int(rng.integers(2, 12))
        a, b = datagen.random_series(rng, 2, L, ("walk", "normal", "int", "const")[t % 4])
        d = oracle_lib.dtw(a, b, L - 1)  # Kim is window-free; DTW_W >= DTW_{L-1}
        assert oracle_lib.lb_kim_sum(a, b) <= d * (1 + 1e-12) + 1e-300


def test_lb_abort_sound(oracle_lib):
    for a, b in rng_pairs(10, 100, 20):
        L = a.size
        w = L // 4
        U, Lo = oracle_lib.envelope(b, w)
        full, _ = oracle_lib.lb_enhanced(a, b, U, Lo, w, 3)
        for D in (0.0, full * 0.5, full, full * 2):
            v, ab = oracle_lib.lb_enhanced(a, b, U, Lo, w, 3, D)
            if ab:
                assert full > D and v == float("inf")
            else:
                assert v == full


def test_nn_exhaustive_vs_bruteforce(oracle_lib):
    rng = np.random.default_rng(11)
    for t in range(6):
        L = int(rng.integers(3, 6))
        T = datagen.random_series(rng, 9, L, ("int", "walk")[t % 2])
        Q = datagen.random_series(rng, 5, L, ("int", "walk")[t % 2])
        T[3] = T[7]  # duplicate -> exact tie, lowest index must win (reading C13)
        w = int(rng.integers(0, L))
        idx, dist = oracle_lib.nn(Q, T, w, mode="exhaustive", threads=2)
        for q in range(Q.shape[0]):
            ds = [brute_dtw(Q[q], T[n], w) for n in range(T.shape[0])]
            bi = min(range(len(ds)), key=lambda n: (ds[n], n))
            assert idx[q] == bi and dist[q] == ds[bi]


@pytest.mark.parametrize("kind", ["walk", "int"])
def test_nn_pruned_equals_exhaustive(oracle_lib, kind):
    rng = np.random.default_rng(12)
    for L, w, V in ((16, 2, 3), (24, 0, 5), (20, 19, 4), (30, 6, 1)):
        T = datagen.random_series(rng, 60, L, kind)
        Q = datagen.random_series(rng, 20, L, kind)
        Q[0] = T[5]
        T[9] = T[40]
        ie, de = oracle_lib.nn(Q, T, w, mode="exhaustive")
        ip, dp, cnt = oracle_lib.nn(Q, T, w, V=V, mode="pruned", with_counts=True)
        assert np.array_equal(ie, ip) and np.array_equal(de, dp)
        assert np.all(cnt["lb_calls"] == T.shape[0])


def test_nn_pruned_on_config0_data(oracle_lib):
    ds = datagen.make_dataset(0)
    w = datagen.window_from_percent(10, 128)
    ie, de = oracle_lib.nn(ds.test[:40], ds.train, w, mode="exhaustive")
    ip, dp, cnt = oracle_lib.nn(ds.test[:40], ds.train, w, V=5, mode="pruned", with_counts=True)
    assert np.array_equal(ie, ip) and np.array_equal(de, dp)
    assert cnt["dtw_calls"].sum() < 40 * 100  # the cascade prunes
    acc = np.mean(ds.train_labels[ie] == ds.test_labels[:40])
    assert acc > 0.8


def test_loocv_vs_bruteforce(oracle_lib):
    rng = np.random.default_rng(13)
    L = 5
    X = datagen.random_series(rng, 10, L, "int")
    X[2] = X[6]
    labels = rng.integers(0, 3, size=10).astype(np.int32)
    windows = [0, 1, 2, 4]
    for mode in ("exhaustive", "pruned"):
        errors, nn = oracle_lib.loocv(X, labels, windows, V=2, mode=mode, threads=2)
        for p, w in enumerate(windows):
            e = 0
            for i in range(10):
                ds = [(brute_dtw(X[i], X[j], w), j) for j in range(10) if j != i]
                bj = min(ds)[1]
                assert nn[p, i] == bj
                e += int(labels[bj] != labels[i])
            assert errors[p] == e


def test_window_rule():
    # reading C4: integer ceil, not float (0.07*300 -> 21, float ceil gives 22)
    assert datagen.window_from_percent(7, 300) == 21
    assert datagen.window_from_percent(10, 128) == 13
    assert datagen.window_from_percent(20, 512) == 103
    assert datagen.window_from_percent(100, 2048) == 2047
    assert [datagen.window_from_percent(p, 256) for p in (1, 10, 20, 50, 100)] == \
        [3, 26, 52, 128, 255]


# ---------------- LB_Improved, LB_New, symmetric LB_Enhanced ----------

def test_next_bounds_hand_example(oracle_lib):
    """Worked by hand (no code): A = (0, 3, 1), B = (1, 0, 2), W = 1.
    Envelope of B (Eq. 3-4): U = (1, 2, 2), L = (0, 0, 0).  LB_Keogh(A,B) = (3-2)^2 = 1.
    Projection: A' = (0, 2, 1); envelope of A': U = (2, 2, 2), L = (0, 0, 1);
    LB_Keogh(B, A') = 0 (B = (1, 0, 2) lies inside), so LB_Improved = 1 + 0 = 1.
    LB_New = delta(0,1) + delta(1,2) + min_{b in {1,0,2}} delta(3,b) = 1 + 1 + 1 = 3.
    DTW_1 by the recurrence: D11=1, D12=1, D21=5, D22=10, D23=2, D32=6, D33=1+min(10,2,6)=3.
    LB_Enhanced^1 (Alg. 1, n_bands=1): 1 + 1 + bridge column 2: (3-2)^2 = 1 -> 3; the reverse
    LB_Enhanced(B,A) with env A = (3,3,3)/(0,0,1): 1 + 1 + 0 = 2 -> symmetric = 3."""
    o = oracle_lib
    A = np.array([0, 3, 1], np.float32)
    B = np.array([1, 0, 2], np.float32)
    assert o.dtw(A, B, 1) == 3.0
    assert o.lb_improved(A, B, 1) == 1.0
    assert o.lb_new(A, B, 1) == 3.0
    assert o.lb_enhanced_sym(A, B, 1, 1) == 3.0
    UA, LA = o.envelope(A, 1)
    assert o.lb_enhanced(B, A, UA, LA, 1, 1)[0] == 2.0


def test_next_bounds_admissible_and_ordered(oracle_lib):
    """Every bound <= DTW_W (brute-force path enumeration, L <= 7, all W); LB_Improved and LB_New
    >= LB_Keogh (both add non-negative terms / take mins over a subset of the envelope range);
    symmetric >= each direction; W = 0 reduces LB_Improved and LB_New to the squared ED;
    LB_New is non-increasing in W (its windows grow)."""
    o = oracle_lib
    for a, b in rng_pairs(21, 120, 7):
        L = a.size
        prev_new = None
        for w in range(0, L):
            d = brute_dtw(a, b, w)
            tol = 1e-12 * max(1.0, d)
            U, Lo = o.envelope(b, w)
            keogh = o.lb_keogh(a, U, Lo)
            imp = o.lb_improved(a, b, w)
            new = o.lb_new(a, b, w)
            assert imp <= d + tol and new <= d + tol, (a, b, w, imp, new, d)
            assert imp >= keogh - tol and new >= keogh - tol
            for V in range(1, L // 2 + 1):
                s = o.lb_enhanced_sym(a, b, w, V)
                f = o.lb_enhanced(a, b, U, Lo, w, V)[0]
                UA, LA = o.envelope(a, w)
                r = o.lb_enhanced(b, a, UA, LA, w, V)[0]
                assert s == max(f, r) and s <= d + tol
            if prev_new is not None:
                assert new <= prev_new + tol
            prev_new = new
        ed = o.sqed(a, b)
        assert o.lb_improved(a, b, 0) == pytest.approx(ed, rel=1e-12, abs=1e-300)
        assert o.lb_new(a, b, 0) == pytest.approx(ed, rel=1e-12, abs=1e-300)


def test_lb_new_is_min_over_window_cells(oracle_lib):
    """LB_New's inner term is the minimum over the band cells of row i: for
    integer series the nearest-value search equals an explicit sort-based nearest neighbour."""
    o = oracle_lib
    rng = np.random.default_rng(23)
    for _ in range(200):
        L = int(rng.integers(3, 30))
        w = int(rng.integers(0, L))
        a, b = datagen.random_series(rng, 2, L, "int")
        tot = (float(a[0]) - float(b[0])) ** 2 + (float(a[-1]) - float(b[-1])) ** 2
        for i in range(1, L - 1):
            win = np.sort(b[max(0, i - w):min(L, i + w + 1)].astype(np.float64))
            k = np.searchsorted(win, float(a[i]))
            cand = [win[j] for j in (k - 1, k) if 0 <= j < win.size]
            tot += min((float(a[i]) - c) ** 2 for c in cand)
        assert o.lb_new(a, b, w) == tot


def test_tightness_hand_example(oracle_lib):
    """oracle.tightness = mean of LB/DTW in the root domain (reading C20: the squared
    values are square-rooted first; pairs with DTW = 0 are excluded).  Worked by hand:
    pairs (lb, dtw^2) = (1,4), (4,16), (9,9), (0,0), (2,8) -> ratios 1/2, 2/4, 3/3, -, 1/2
    -> mean 2.5/4 = 0.625 over 4 pairs.  Without the square roots the mean would be 0.4375;
    counting the DTW = 0 pair would change the count to 5."""
    t, n = oracle_lib.tightness([1, 4, 9, 0, 2], [4, 16, 9, 0, 8])
    assert n == 4
    assert t == 0.625


def test_tightness_special_cases(oracle_lib):
    """At W = 0 the envelope of B is B itself, so LB_Keogh = squared ED = DTW_0:
    tightness exactly 1 on pairs with distinct series; any admissible bound gives <= 1."""
    rng = np.random.default_rng(37)
    X = datagen.random_series(rng, 12, 40, "walk")
    lb = [oracle_lib.lb_keogh(X[i], X[i + 6], X[i + 6]) for i in range(6)]
    d = [oracle_lib.dtw(X[i], X[i + 6], 0) for i in range(6)]
    t, n = oracle_lib.tightness(lb, d)
    assert n == 6 and abs(t - 1.0) < 1e-12
    w = 5
    U, Lo = oracle_lib.envelopes(X, w)
    lb = [oracle_lib.lb_enhanced(X[i], X[i + 6], U[i + 6], Lo[i + 6], w, 3)[0] for i in range(6)]
    d = [oracle_lib.dtw(X[i], X[i + 6], w) for i in range(6)]
    t, n = oracle_lib.tightness(lb, d)
    assert n == 6 and 0.0 < t <= 1.0


def test_enhanced_improved_admissible_and_dominant(oracle_lib):
    """LB_Enhanced^V with the LB_Improved bridge (reading C21): <= DTW_W (brute-force
    path enumeration, L <= 8, every W and V), >= LB_Enhanced^V (it adds non-negative terms),
    equal to it at W = 0 (A' = B, so env A' = B) and when the bridge is empty (V >= L/2), and
    strictly tighter on some pairs (the second pass is live)."""
    o = oracle_lib
    strict = 0
    for a, b in rng_pairs(42, 90, 8, kinds=("walk", "normal")):
        L = a.size
        for w in range(0, L):
            d = brute_dtw(a, b, w)
            tol = 1e-12 * max(1.0, d)
            U, Lo = o.envelope(b, w)
            for V in range(1, L // 2 + 1):
                e = o.lb_enhanced(a, b, U, Lo, w, V)[0]
                ei = o.lb_enhanced_improved(a, b, w, V)
                assert ei <= d + tol, (a, b, w, V, ei, d)
                assert ei >= e - tol
                if w == 0 or 2 * min(L // 2, V) >= L:
                    assert ei == e
                strict += ei > e * (1 + 1e-9) + 1e-12
    assert strict > 50
    # larger series against the (pinned) DP DTW
    rng = np.random.default_rng(43)
    X = datagen.random_series(rng, 40, 64, "walk")
    for i in range(20):
        for w in (1, 3, 6, 20, 63):
            d = o.dtw(X[i], X[i + 20], w)
            for V in (1, 3, 5, 16):
                assert o.lb_enhanced_improved(X[i], X[i + 20], w, V) <= d * (1 + 1e-12)


def test_loocv_degenerate_sizes(oracle_lib):
    # reading C17: with one series there is no other candidate (index -1, counted as an error);
    # with two, each is the other's neighbour whatever the window
    rng = np.random.default_rng(21)
    X = datagen.random_series(rng, 2, 16, "walk")
    for mode in ("exhaustive", "pruned"):
        err, nn = oracle_lib.loocv(X[:1], np.array([3], np.int32), [0, 4, 15], mode=mode)
        assert (nn == -1).all() and (err == 1).all()
        err, nn = oracle_lib.loocv(X, np.array([3, 4], np.int32), [0, 4, 15], mode=mode)
        assert (nn == [[1, 0]] * 3).all() and (err == 2).all()
        err, nn = oracle_lib.loocv(X, np.array([3, 3], np.int32), [0, 4, 15], mode=mode)
        assert (nn == [[1, 0]] * 3).all() and (err == 0).all()
