"""Tightness of the lower bounds on config 1 (the paper's Fig. 1/2
analogue on synthetic pairs): mean sqrt(LB)/DTW over all N x Q = 1e6 pairs per
window, with each bound's all-pairs kernel time on one B200.

  python tools/tightness.py [--out profiles/round1_tightness.md] [--n 1000]

Every number comes from the library's kernels (bounds, all-pairs DTW via nndtw_dtw_batch,
the tightness reduction via nndtw_tightness).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=1000)
    args = ap.parse_args()
    ds = datagen.make_dataset(1, n_train=args.n, n_test=args.n)
    q = torch.as_tensor(ds.test, device="cuda")
    t = torch.as_tensor(ds.train, device="cuda")
    nq, nt = q.shape[0], t.shape[0]
    ia = torch.arange(nq, device="cuda", dtype=torch.int32).repeat_interleave(nt)
    ib = torch.arange(nt, device="cuda", dtype=torch.int32).repeat(nq)
    rows = []
    Vs = (1, 2, 4, 5, 8)
    for p in ds.cfg.percents:
        w = datagen.window_from_percent(p, ds.cfg.L)
        d, ms_dtw = timed(lambda: nndtw.dtw_batch(q, t, w, ia, ib))
        U, Lo, kim = nndtw.envelopes(t, w)
        qenv = nndtw.envelopes(q, w)
        bounds = {"LB_Keogh": lambda: nndtw.lb_enhanced(q, t, U, Lo, w, 1, keogh=True)}
        for V in Vs:
            bounds[f"LB_Enhanced^{V}"] = (lambda V=V: nndtw.lb_enhanced(q, t, U, Lo, w, V))
        bounds["LB_Enhanced^5 symmetric"] = lambda: nndtw.lb_enhanced_symmetric(
            q, t, w, 5, q_env=qenv, t_env=(U, Lo, kim))
        bounds["LB_Improved"] = lambda: nndtw.lb_improved(q, t, w, t_env=(U, Lo))
        bounds["LB_New"] = lambda: nndtw.lb_new(q, t, w)
        for name, fn in bounds.items():
            lb, ms = timed(fn)
            mean, cnt, mx = nndtw.tightness(lb, d)
            rows.append({"p": p, "w": w, "bound": name, "tightness": mean, "pairs": cnt,
                         "max_ratio": mx, "ms": ms, "dtw_ms": ms_dtw})
            print(json.dumps(rows[-1]), flush=True)
    if args.out:
        names = list(dict.fromkeys(r["bound"] for r in rows))
        ws = list(dict.fromkeys((r["p"], r["w"]) for r in rows))
        by = {(r["p"], r["bound"]): r for r in rows}
        lines = [f"# Tightness on config 1 ({nq} x {nt} pairs, L={ds.cfg.L}), one B200\n",
                 "Mean sqrt(LB) / DTW over all pairs with DTW > 0 (P:37; reading C20), from the "
                 "library's kernels (`tools/tightness.py`); the Fig. 1/2 analogue on synthetic "
                 "pairs (the UCR archive is not available, P:560).  Max ratio <= 1 everywhere "
                 "(admissibility).  Second table: all-pairs kernel time per bound (ms).\n",
                 "| bound | " + " | ".join(f"W={p}% (w={w})" for p, w in ws) + " |",
                 "|---|" + "---|" * len(ws)]
        for nm in names:
            lines.append(f"| {nm} | " + " | ".join(f"{by[(p, nm)]['tightness']:.4f}"
                                                     for p, _ in ws) + " |")
        lines += ["", "| bound (ms, all pairs) | " + " | ".join(f"w={w}" for _, w in ws) + " |",
                  "|---|" + "---|" * len(ws)]
        for nm in names:
            lines.append(f"| {nm} | " + " | ".join(f"{by[(p, nm)]['ms']:.2f}" for p, _ in ws)
                         + " |")
        lines.append("| DTW (exhaustive, for reference) | " +
                     " | ".join(f"{by[(p, names[0])]['dtw_ms']:.2f}" for p, _ in ws) + " |")
        lines.append("\nmax ratio over all bounds and windows: "
                     f"{max(r['max_ratio'] for r in rows):.6f}")
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")
        with open(os.path.splitext(args.out)[0] + ".jsonl", "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
