"""V-sweep (the shape of the paper's Fig. 9) on BJ:configs[1]:
NN-DTW time with LB_Kim -> LB_Enhanced^V normalised by the same pipeline with LB_Kim -> LB_Keogh,
per window.  Also the DTW-work ratio (cells evaluated), which does not depend on the hardware.
Envelopes are precomputed and not timed.  Synthetic data (datagen), one B200.

    python tools/vsweep.py [--reps 5] [--out profiles/round1_vsweep.md]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402

VS = [1, 2, 3, 4, 5, 6, 8, 10, 12, 15, 20]


def run(model, q, reps):
    nndtw.classify(model, q, check=False)
    ts = []
    st = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pred = nndtw.classify(model, q, stats=True, check=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        st = pred.stats
    return float(np.median(ts)), st, pred.idx.cpu().numpy()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ds = datagen.make_dataset(1)
    dev = torch.device("cuda")
    tr = torch.as_tensor(ds.train, device=dev)
    te = torch.as_tensor(ds.test, device=dev)
    lab = torch.as_tensor(ds.train_labels, device=dev)
    lines = ["| W (% of L) | w | Keogh ms | " + " | ".join(f"V={v}" for v in VS) + " |",
             "|---|---|---|" + "---|" * len(VS)]
    wl = ["| W | w | Keogh cells | " + " | ".join(f"V={v}" for v in VS) + " |",
          "|---|---|---|" + "---|" * len(VS)]
    for p in ds.cfg.percents:
        w = datagen.window_from_percent(p, 256)
        mk = nndtw.Model(tr, lab, w, 5, check=False, bound="keogh")
        tk, sk, ik = run(mk, te, args.reps)
        row, rw = [], []
        for v in VS:
            me = nndtw.Model(tr, lab, w, v, check=False)
            te_, se, ie = run(me, te, args.reps)
            assert np.array_equal(ie, ik), "bounds disagree on the exact answer"
            row.append(f"{te_ / tk:.3f}")
            rw.append(f"{(se['cells'] + 1) / (sk['cells'] + 1):.3f}")
        lines.append(f"| {p} | {w} | {tk:.3f} | " + " | ".join(row) + " |")
        wl.append(f"| {p} | {w} | {sk['cells']:.3g} | " + " | ".join(rw) + " |")
        print(lines[-1], flush=True)
    txt = ("# V-sweep on config 1 (N=Q=1000, L=256), one B200\n\n"
           "NN-DTW time (S2-S7, envelopes precomputed) with LB_Kim -> LB_Enhanced^V divided by "
           "the same pipeline with LB_Kim -> LB_Keogh; < 1 means LB_Enhanced^V is faster "
           "(cf. the paper's Fig. 9, P:577-612).\n\n" + "\n".join(lines) +
           "\n\nDTW work (in-band cells evaluated) relative to LB_Keogh:\n\n" + "\n".join(wl) + "\n")
    if args.out:
        open(args.out, "w").write(txt)
    print(txt)


if __name__ == "__main__":
    main()
