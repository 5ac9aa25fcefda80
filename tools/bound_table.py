"""NN-DTW classification time per S2 bound (the paper's Fig. 9-11 comparison, on the
synthetic configs).

For each window and each bound -- LB_Keogh, LB_Enhanced^V (V = 5), LB_Improved (O(L) projection
envelopes), LB_New, LB_Enhanced^5 with the LB_Improved bridge, the symmetric LB_Enhanced^5, and no
bound at all (DTW with early abandoning only) -- classify every query (config 1) or a query
subset (config 2) through nndtw.classify, CUDA-event timed (median of reps, after a warm-up), and
report the time normalised by LB_Keogh's, the S2 / S4 split, DTW calls and cells.  Every bound
must give the same answer (checked here against the first bound's).

  python tools/bound_table.py [--config 1|2] [--queries N] [--reps 3] > profiles/<tag>.md
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402

BOUNDS = [("LB_Keogh", dict(bound="keogh")),
          ("LB_Enhanced^5", dict(bound="enhanced")),
          ("LB_Improved", dict(bound="improved")),
          ("LB_New", dict(bound="new")),
          ("LB_Enh^5+Improved bridge", dict(bound="enhanced_improved")),
          ("symmetric LB_Enh^5", dict(bound="enhanced", symmetric=True)),
          ("no bound", dict(bound="none"))]


def run(model, q, reps):
    nndtw.classify(model, q, check=False)
    torch.cuda.synchronize()
    ts, st = [], None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p = nndtw.classify(model, q, check=False, stats=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        st = p.stats
    return float(np.median(ts)), st, p.idx.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--queries", type=int, default=None)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--skip", default="", help="comma-separated bound names to skip")
    a = ap.parse_args()
    ds = datagen.make_dataset(a.config)
    Q = ds.test if a.queries is None else ds.test[:a.queries]
    dev = torch.device("cuda:0")
    t = torch.as_tensor(ds.train, device=dev)
    lab = torch.as_tensor(ds.train_labels, device=dev)
    q = torch.as_tensor(Q, device=dev)
    windows = ds.cfg.windows() if a.config == 1 else [ds.cfg.windows()[0]]
    skip = set(s for s in a.skip.split(",") if s)
    print(f"# NN-DTW time per bound, config {a.config} (N={t.shape[0]}, Q={q.shape[0]}, "
          f"L={t.shape[1]}, V=5), one B200\n")
    print("Classification time of S2-S7 (nndtw.classify, stats on), median of "
          f"{a.reps} after a warm-up; envelopes precomputed (P:583).  ratio = time / LB_Keogh's "
          "(the paper's normalisation, Fig. 9).\n")
    print("| w | bound | ms | ratio | S2 ms | S4 ms | survivors | DTW calls | cells |")
    print("|---|---|---|---|---|---|---|---|---|")
    for w in windows:
        base, ref = None, None
        for name, kw in BOUNDS:
            if name in skip:
                continue
            model = nndtw.Model(t, lab, w, 5, **kw)
            ms, st, idx = run(model, q, a.reps)
            if ref is None:
                ref = idx
            assert np.array_equal(idx, ref), f"{name}: different answer"
            base = base or ms
            print(f"| {w} | {name} | {ms:.3f} | {ms / base:.2f} | {st['ms_lb']:.3f} | "
                  f"{st['ms_dtw']:.3f} | {st['survivors']} | {st['dtw_calls']} | "
                  f"{st['cells']:.3g} |", flush=True)
            del model
    print("\nEvery bound returned the same neighbours (asserted).")


if __name__ == "__main__":
    main()
