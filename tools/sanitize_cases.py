"""Small inputs that launch every kernel of libnndtw.so, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck -- one tool per run, SURVEY.md §5 "race detection"):

  compute-sanitizer --tool racecheck --error-exitcode 99 python tools/sanitize_cases.py

Covered: S1 envelopes (direct kernel for every residue class used, van Herk kernel), Kim
stats, the S2 tile kernel and the two-stage S2 (column compaction, sparse bridge) (LB_Enhanced with/without Kim, LB_Keogh, symmetric, level counts, V
above the shared-memory band limit), LB_Improved / LB_Enhanced+Improved / LB_New, the bound
finish pass, every band-kernel layout class (aligned full-warp KM=2 with and without packing,
aligned KM=1, general KM=0, R = 32), the strip kernel with KS = 1 / 2 / 4 (masked and full
window), the w = 0 kernel, S3 compaction / seeds / bucket scan, S7 refine / resolve / overflow,
S8 LOOCV, the sharded phases, tightness and the finite check.  Prints one line per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402

dev = torch.device("cuda:0")


def T(x):
    return torch.as_tensor(np.ascontiguousarray(x), device=dev)


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    print("library", nndtw.LIB_PATH, flush=True)
    rng = np.random.default_rng(5)
    # S0-S7 on config 0 (all of classify's kernels), with stats and level counts
    ds = datagen.make_dataset(0)
    w0 = ds.cfg.windows()[0]
    model = nndtw.Model(T(ds.train), T(ds.train_labels), w0, 5)
    case("classify config 0 (+level stats)",
         lambda: nndtw.classify(model, T(ds.test[:40]), stats=True, level_stats=True))
    for bound in ("keogh", "improved", "new", "enhanced_improved", "none"):
        m = nndtw.Model(T(ds.train), T(ds.train_labels), w0, 5, bound=bound)
        case(f"classify bound={bound}", lambda m=m: nndtw.classify(m, T(ds.test[:24]), stats=True,
                                                                    level_stats=True))
    # the two-stage S2 (stage A tile, column compaction + scan, sparse bridge, second seed)
    os.environ["NNDTW_S2_STAGES"] = "2"
    case("classify two-stage S2", lambda: nndtw.classify(model, T(ds.test[:40]), stats=True))
    d1 = datagen.make_dataset(1, n_train=300, n_test=40)
    m1 = nndtw.Model(T(d1.train), T(d1.train_labels), d1.cfg.windows()[0], 5)
    case("classify two-stage S2 L=256", lambda: nndtw.classify(m1, T(d1.test)))
    del os.environ["NNDTW_S2_STAGES"]
    # config 2's band layout (R = 26, full warp): the survivor round's padded query copy (GA)
    d2 = datagen.make_dataset(2, n_train=300, n_test=32)
    m2 = nndtw.Model(T(d2.train), T(d2.train_labels), d2.cfg.windows()[0], 5)
    case("classify L=512 w=103 (GA band variant)", lambda: nndtw.classify(m2, T(d2.test)))
    ms = nndtw.Model(T(ds.train), T(ds.train_labels), w0, 5, symmetric=True)
    case("classify symmetric", lambda: nndtw.classify(ms, T(ds.test[:24])))

    # sharded phases (seed / search / search_a / search_b) and the fp64 refine / resolve
    def sharded():
        q = T(ds.test[:24])
        for phases in (("seed", "search"), ("seed", "search_a", "search_b")):
            key, ws, _ = nndtw.classify_keys(model, q, exact=False, phase="seed")
            for ph in phases[1:]:
                key, ws, _ = nndtw.classify_keys(model, q, exact=False, phase=ph, key=key, ws=ws)
            f64 = nndtw.classify_refine(model, q, ws, key)
            nndtw.classify_resolve(model, q, ws, key, f64)
    case("sharded phases + refine/resolve", sharded)

    # tie-log overflow path (refine_overflow)
    os.environ["NNDTW_TIE_LOG_CAP"] = "3"
    Tr = datagen.random_series(rng, 60, 24, "int")
    Tr = np.concatenate([Tr, Tr])
    mt = nndtw.Model(T(Tr), T(np.arange(120, dtype=np.int32)), 3, 3)
    case("classify tie-log overflow", lambda: nndtw.classify(mt, T(Tr[:20])))
    del os.environ["NNDTW_TIE_LOG_CAP"]

    # S1: van Herk (w < 16 / long windows) and the direct kernel over residues R = w mod 16
    for L, ws in ((64, (0, 3, 15)), (300, (16, 17, 23, 31, 45, 60, 299)), (512, (103, 40)),
                  (2048, (2047, 409))):
        X = T(datagen.random_series(rng, 9, L, "walk"))
        for w in ws:
            case(f"envelopes L={L} w={w}", lambda X=X, w=w: nndtw.envelopes(X, w))

    # S2 variants
    Q = T(datagen.random_series(rng, 70, 256, "walk"))
    Tn = T(datagen.random_series(rng, 130, 256, "walk"))
    U, Lo, kim = nndtw.envelopes(Tn, 26)
    case("lb_enhanced +kim", lambda: nndtw.lb_enhanced(Q, Tn, U, Lo, 26, 5, True, None, kim))
    case("lb_enhanced V=40 (global band reads)", lambda: nndtw.lb_enhanced(Q, Tn, U, Lo, 26, 40))
    case("lb_keogh", lambda: nndtw.lb_enhanced(Q, Tn, U, Lo, 26, 5, keogh=True))
    case("lb symmetric", lambda: nndtw.lb_enhanced_symmetric(Q, Tn, 26, 5, with_kim=True))
    case("lb_improved", lambda: nndtw.lb_improved(Q, Tn, 26))
    case("lb_enhanced_improved", lambda: nndtw.lb_enhanced_improved(Q, Tn, 26, 5))
    case("lb_new", lambda: nndtw.lb_new(Q[:8], Tn[:16], 26))

    # S4 band layouts (dtw_batch, with cutoffs so that abandoning runs too)
    def dtw(L, w, n=40):
        A = T(datagen.random_series(rng, n, L, "walk"))
        B = T(datagen.random_series(rng, n, L, "walk"))
        full = nndtw.dtw_batch(A, B, w)
        nndtw.dtw_batch(A, B, w, cutoff=full * 0.7)
    for L, w in ((512, 103), (256, 26), (256, 52), (300, 60), (300, 150), (300, 192), (300, 225),
                 (1024, 511), (128, 127), (64, 0), (300, 0)):
        case(f"dtw band/w0 L={L} w={w}", lambda L=L, w=w: dtw(L, w))
    # S4 strip kernel: KS = 1 (L < 512), 2 (512 <= L < 1024), 4 (L >= 1024); masked and full
    for L, w in ((256, 255), (300, 299), (600, 599), (600, 520), (1024, 1023), (2048, 2047),
                 (2048, 1500)):
        case(f"dtw strip L={L} w={w}", lambda L=L, w=w: dtw(L, w, 12))

    # S8 LOOCV (reduced) and the tightness reduction
    d3 = datagen.make_dataset(3, n_train=80)
    case("loocv", lambda: nndtw.loocv_window(T(d3.train), T(d3.train_labels), [0, 3, 30, 299],
                                             v=5, with_nn=True, stats=True))
    lbm = nndtw.lb_enhanced(Q[:10], Tn[:20], U[:20], Lo[:20], 26, 5)
    dd = torch.rand(200, device=dev) + 1.0
    case("tightness", lambda: nndtw.tightness(lbm, dd))
    case("check_finite", lambda: nndtw.check_finite(Q))
    print("all sanitizer cases done", flush=True)


if __name__ == "__main__":
    main()
