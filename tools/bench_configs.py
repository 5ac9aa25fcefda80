"""Time the hot path on every BASELINE.json config (one GPU), for BASELINE.md's table.

  python tools/bench_configs.py [--configs 0,1,3,4] [--reps 3]

Per config: queries/s over S1-S7 (envelopes included), DTW GCUPS (survivor round), counters.
Config 1 is the 25-point (W, V) grid; config 3 is the 101-window leave-one-out search
(windows/s and per-window error counts).  Device time via CUDA events, median of reps.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402


def timed(fn, reps):
    out = []
    res = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res = fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out)), res


def classify_cfg(ds, w, V, reps):
    dev = torch.device("cuda")
    tr = torch.as_tensor(ds.train, device=dev)
    te = torch.as_tensor(ds.test, device=dev)
    lab = torch.as_tensor(ds.train_labels, device=dev)

    def step():
        m = nndtw.Model(tr, lab, w, V, check=False)
        return nndtw.classify(m, te, stats=True, check=False)

    step()
    ms, pred = timed(step, reps)
    st = pred.stats
    acc = float((pred.label.cpu().numpy() == ds.test_labels).mean())
    Q, N, L = ds.test.shape[0], ds.train.shape[0], ds.train.shape[1]
    # S2-S7 only (envelopes precomputed), eager and as one CUDA-graph replay
    model = nndtw.Model(tr, lab, w, V, check=False)
    ms_s2, _ = timed(lambda: nndtw.classify(model, te, check=False), reps)
    g = nndtw.GraphedClassifier(model, Q)
    ms_graph, _ = timed(lambda: g(te), max(reps, 5))
    return {"Q": Q, "N": N, "L": L, "w": w, "V": V, "ms": ms, "queries_s": Q / (ms / 1e3),
            "ms_s2s7": ms_s2, "ms_s2s7_graph": ms_graph,
            "queries_s_graph": Q / (ms_graph / 1e3),
            "dtw_gcups": st["cells"] / (st["ms_dtw"] * 1e-3) / 1e9 if st["ms_dtw"] else 0,
            "ms_lb": st["ms_lb"], "ms_dtw": st["ms_dtw"], "ms_other": st["ms_other"],
            "survivor_frac": st["survivors"] / max(1, st["lb_pairs"]),
            "dtw_calls": st["dtw_calls"], "cells": st["cells"], "accuracy": acc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,3,4")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    rows = []
    for c in [int(x) for x in args.configs.split(",")]:
        cfg = datagen.CONFIGS[c]
        ds = datagen.make_dataset(c)
        if c == 3:
            dev = torch.device("cuda")
            x = torch.as_tensor(ds.train, device=dev)
            lab = torch.as_tensor(ds.train_labels, device=dev)
            wins = cfg.windows()
            nndtw.loocv_window(x, lab, wins[:3], v=5)
            ms, (err, _, st) = timed(lambda: nndtw.loocv_window(x, lab, wins, v=5, stats=True),
                                     max(1, args.reps - 1))
            e = err.cpu().numpy()
            gl = nndtw.GraphedLoocv(x, lab, wins, v=5)
            ms_g, _ = timed(gl, max(1, args.reps - 1))
            rows.append({"config": 3, "N": cfg.n_train, "L": cfg.L, "windows": len(wins),
                         "ms": ms, "windows_s": len(wins) / (ms / 1e3), "ms_graph": ms_g,
                         "windows_s_graph": len(wins) / (ms_g / 1e3),
                         "heldout_queries_s": len(wins) * cfg.n_train / (ms / 1e3),
                         "best_w": int(wins[int(np.argmin(e))]), "min_errors": int(e.min()),
                         "errors_first": e[:8].tolist(), "dtw_calls": st["dtw_calls"],
                         "cells": st["cells"]})
        else:
            grid = [(w, V) for w in cfg.windows() for V in cfg.Vs] if c == 1 else \
                [(cfg.windows()[0], cfg.Vs[-1])]
            for w, V in grid:
                r = classify_cfg(ds, w, V, args.reps)
                r["config"] = c
                rows.append(r)
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"all": rows}))


if __name__ == "__main__":
    main()
