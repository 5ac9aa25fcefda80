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
        for mode in ("own", "seed", "split"):
            if G == 1 and mode != "own":
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

            def timed(fn):
                e0 = ev()
                out = fn()
                e1 = ev()
                torch.cuda.synchronize()
                return out, e0.elapsed_time(e1)

            def gmin(keys):
                g = keys[0].clone()
                for k in keys[1:]:
                    g = torch.minimum(g, k)
                return g

            seeds, t_seed = [], []
            for m in models:
                out, t = timed(lambda: nndtw.classify_keys(m, q, exact=False, stats=True,
                                                           phase="seed"))
                seeds.append(out)
                t_seed.append(t)
            gseed = gmin([k for k, _, _ in seeds])
            phase_ms = [max(t_seed)]
            st_all = [st for _, _, st in seeds]
            if mode == "split":
                mids, t_a = [], []
                for m, (k, ws, st) in zip(models, seeds):
                    out, t = timed(lambda: nndtw.classify_keys(
                        m, q, exact=False, stats=True, phase="search_a", key=gseed.clone(),
                        ws=ws))
                    mids.append(out)
                    t_a.append(t)
                gmid = gmin([k for k, _, _ in mids])
                t_b = []
                for i, (m, (k, ws, st)) in enumerate(zip(models, seeds)):
                    (_, _, st2), t = timed(lambda: nndtw.classify_keys(
                        m, q, exact=False, stats=True, phase="search_b", key=gmid.clone(),
                        ws=ws))
                    t_b.append(t)
                    st_all[i] = nndtw.merge_stats(nndtw.merge_stats(st_all[i], mids[i][2]), st2)
                phase_ms += [max(t_a), max(t_b)]
            else:
                t_s = []
                for i, (m, (k, ws, st)) in enumerate(zip(models, seeds)):
                    start = gseed.clone() if mode == "seed" else k
                    (_, _, st2), t = timed(lambda: nndtw.classify_keys(
                        m, q, exact=False, stats=True, phase="search", key=start, ws=ws))
                    t_s.append(t)
                    st_all[i] = nndtw.merge_stats(st_all[i], st2)
                phase_ms += [max(t_s)]
            step = sum(phase_ms)  # the all-reduces between phases synchronise the shards
            row = {"gpus": G, "exchange": mode, "step_ms": step,
                   "phase_ms": [round(x, 2) for x in phase_ms],
                   "cells": sum(s["cells"] for s in st_all),
                   "dtw_calls": sum(s["dtw_calls"] for s in st_all),
                   "queries_s_projected": q.shape[0] / (step / 1e3)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        base = rows[0]["step_ms"]
        lines = ["# Projected multi-GPU scaling of config 2 (one B200, shards run in turn)\n",
                 "Each shard runs its S2-S5 work on its contiguous train slice (dist.py), phase by "
                 "phase; a G-GPU step is the sum over phases of the slowest shard (the Q x 8-byte "
                 "MIN all-reduces between phases synchronise the ranks; their tens of "
                 "microseconds on NVLink are not included).  Exchange 'own': every shard prunes "
                 "against its own seed; 'seed': against the MIN over shards of the seed keys "
                 "(NNDTW_CLASSIFY_PHASE_SEED / _SEARCH; dist.py's default, split=False); 'split': "
                 "in addition the survivor round runs in two halves with another MIN between "
                 "them (PHASE_SEARCH_A / _B; dist.py with split=True).\n",
                 "| GPUs | exchange | step ms (phases) | projected queries/s | "
                 "projected efficiency | DTW cells (all shards) | DTW calls |",
                 "|---|---|---|---|---|---|---|"]
        for r in rows:
            eff = base / (r["step_ms"] * r["gpus"])
            ph = " + ".join(f"{x:.1f}" for x in r["phase_ms"])
            lines.append(f"| {r['gpus']} | {r['exchange']} | {r['step_ms']:.1f} ({ph}) | "
                         f"{r['queries_s_projected']:.0f} | {eff:.2f} | {r['cells']:.3e} | "
                         f"{r['dtw_calls']:.3e} |")
        with open(args.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
