"""Projected multi-GPU behaviour on one B200: config 2's train set split into G contiguous
shards, each shard's hot path run in turn (seed phase, MIN of the seed keys, search phase), as
dist.py runs them on G GPUs.  Reports per shard the device time of its S2-S5 work and its DTW
cells; max over shards = the time a G-GPU step would take (collectives excluded, ~tens of us).

  python tools/shard_sim.py [--gpus 1,2,4,8] [--no-global-seed] [--out profiles/...md]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402
from paper_1808_09617_b200.dist import shard_range  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ds = datagen.make_dataset(2)
    w, V = ds.cfg.windows()[0], 5
    tr = torch.as_tensor(ds.train, device="cuda")
    lab = torch.as_tensor(ds.train_labels, device="cuda")
    q = torch.as_tensor(ds.test, device="cuda")
    N = tr.shape[0]
    rows = []
    for G in [int(x) for x in args.gpus.split(",")]:
        for glob in (False, True):
            if G == 1 and glob:
                continue
            models = []
            for r in range(G):
                lo, hi = shard_range(N, r, G)
                models.append(nndtw.Model(tr[lo:hi].contiguous(), lab[lo:hi], w, V,
                                          index_base=lo, check=False))
            # warm-up
            for m in models:
                nndtw.classify_keys(m, q, exact=False)
            torch.cuda.synchronize()
            t_seed, t_search, st_all = [], [], []
            seeds = []
            for m in models:
                e0 = ev()
                k, ws, st = nndtw.classify_keys(m, q, exact=False, stats=True, phase="seed")
                e1 = ev()
                torch.cuda.synchronize()
                t_seed.append(e0.elapsed_time(e1))
                seeds.append((k, ws, st))
            gseed = seeds[0][0].clone()
            for k, _, _ in seeds[1:]:
                gseed = torch.minimum(gseed, k)
            for m, (k, ws, st) in zip(models, seeds):
                start = gseed.clone() if glob else k
                e0 = ev()
                _, _, st2 = nndtw.classify_keys(m, q, exact=False, stats=True, phase="search",
                                                key=start, ws=ws)
                e1 = ev()
                torch.cuda.synchronize()
                t_search.append(e0.elapsed_time(e1))
                st_all.append(nndtw.merge_stats(st, st2))
            per = [a + b for a, b in zip(t_seed, t_search)]
            row = {"gpus": G, "global_seed": glob, "max_shard_ms": max(per),
                   "sum_shard_ms": sum(per), "cells": sum(s["cells"] for s in st_all),
                   "dtw_calls": sum(s["dtw_calls"] for s in st_all),
                   "queries_s_projected": q.shape[0] / (max(per) / 1e3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        base = rows[0]["max_shard_ms"]
        lines = ["# Projected multi-GPU scaling of config 2 (one B200, shards run in turn)\n",
                 "Each shard runs its S2-S5 work on its contiguous train slice (dist.py); the "
                 "projected G-GPU step time is the slowest shard (the three Q x 8-byte MIN "
                 "all-reduces, tens of microseconds on NVLink, are not included).  'global "
                 "seed': shards prune against the MIN over shards of the seed keys "
                 "(NNDTW_CLASSIFY_PHASE_SEED / _SEARCH); otherwise each against its own seed.\n",
                 "| GPUs | global seed | slowest shard ms | projected queries/s | "
                 "projected efficiency | DTW cells (all shards) | DTW calls |",
                 "|---|---|---|---|---|---|---|"]
        for r in rows:
            eff = base / (r["max_shard_ms"] * r["gpus"])
            lines.append(f"| {r['gpus']} | {'yes' if r['global_seed'] else 'no'} | "
                         f"{r['max_shard_ms']:.1f} | {r['queries_s_projected']:.0f} | "
                         f"{eff:.2f} | {r['cells']:.3e} | {r['dtw_calls']:.3e} |")
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
