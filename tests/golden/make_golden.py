"""Write the full-size oracle answers of BASELINE.json configs 0-4 to tests/golden/cfg{k}.npz.

Imports only `oracle/` (the fp64 CPU oracle) and `datagen.py` (seeded inputs, no method
arithmetic): no expected value here comes from the CUDA path.  The -m gpu test
`tests/test_gpu_golden.py` compares EVERY query of every config against these files
(north_star: results identical to the oracle on all five configs; pruning is lossless by
Thm 2, so the exact 1-NN under lowest-index ties, P:58 / reading C13, is the answer).

Per config:
  cfg0        idx[Q], dist[Q] (fp64 squared DTW), label[Q]            -- exhaustive mode (i)
  cfg1        idx_w{w}[Q], dist_w{w}[Q], label_w{w}[Q] for the 5 windows -- pruned mode (ii)
  cfg2, cfg4  idx[Q], dist[Q], label[Q]                               -- pruned mode (ii)
  cfg3        errors[101], nn[101][2000] (leave-one-out, reading C17)  -- pruned mode (ii)
Mode (ii) is the paper's sequential search (ED order P:569, Alg. 1 with the abort, DTW with
abandoning); it is pinned to mode (i) in tests/test_oracle_pins.py.

The large configs take hours on 8 cores, so they are computed in query chunks that are
checkpointed under tests/golden/.partial/ (resumable; deleted once the file is complete).

    python tests/golden/make_golden.py [--configs 0 1 3 2 4] [--threads N] [--chunk 256]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle   # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
PARTIAL = os.path.join(GOLDEN, ".partial")


def _log(msg):
    print(time.strftime("%H:%M:%S"), msg, flush=True)


def _chunked_nn(tag, Q, T, w, V, threads, chunk):
    """oracle.nn in checkpointed query chunks; returns (idx int64, dist f64)."""
    os.makedirs(PARTIAL, exist_ok=True)
    U, Lo = oracle.envelopes(T, w)
    idx = np.empty(Q.shape[0], np.int64)
    dist = np.empty(Q.shape[0], np.float64)
    for s in range(0, Q.shape[0], chunk):
        e = min(Q.shape[0], s + chunk)
        f = os.path.join(PARTIAL, f"{tag}_{s}_{e}.npz")
        if os.path.exists(f):
            z = np.load(f)
            idx[s:e], dist[s:e] = z["idx"], z["dist"]
            continue
        t0 = time.time()
        i, d = oracle.nn(Q[s:e], T, w, V=V, mode="pruned", threads=threads,
                         envelopes_UL=(U, Lo))
        np.savez(f, idx=i, dist=d)
        idx[s:e], dist[s:e] = i, d
        _log(f"{tag} queries [{s},{e}) {time.time() - t0:.1f} s")
    return idx, dist


def golden_cfg(c, threads, chunk):
    out = os.path.join(GOLDEN, f"cfg{c}.npz")
    if os.path.exists(out):
        _log(f"{out} exists, skipped")
        return
    t0 = time.time()
    ds = datagen.make_dataset(c)
    cfg = ds.cfg
    V = cfg.Vs[-1] if c == 4 else 5
    res = {"L": np.int64(cfg.L)}
    if c == 0:
        w = cfg.windows()[0]
        i, d = oracle.nn(ds.test, ds.train, w, mode="exhaustive", threads=threads)
        res.update(w=np.int64(w), idx=i, dist=d, label=ds.train_labels[i])
    elif c == 1:
        ws = cfg.windows()
        res["windows"] = np.array(ws, np.int64)
        for w in ws:
            i, d = _chunked_nn(f"cfg1_w{w}", ds.test, ds.train, w, V, threads, chunk)
            res[f"idx_w{w}"], res[f"dist_w{w}"] = i, d
            res[f"label_w{w}"] = ds.train_labels[i]
    elif c in (2, 4):
        w = cfg.windows()[0]
        i, d = _chunked_nn(f"cfg{c}", ds.test, ds.train, w, V, threads, chunk)
        res.update(w=np.int64(w), V=np.int64(V), idx=i, dist=d, label=ds.train_labels[i])
    elif c == 3:
        ws = cfg.windows()
        n = ds.train.shape[0]
        errors = np.zeros(len(ws), np.int64)
        nn = np.empty((len(ws), n), np.int64)
        os.makedirs(PARTIAL, exist_ok=True)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            f = os.path.join(PARTIAL, f"cfg3_{s}_{e}.npz")
            if os.path.exists(f):
                z = np.load(f)
                nn[:, s:e] = z["nn"]
                continue
            t1 = time.time()
            _, part = oracle.loocv(ds.train, ds.train_labels, ws, V=V, q_begin=s, q_end=e,
                                   mode="pruned", threads=threads)
            np.savez(f, nn=part)
            nn[:, s:e] = part
            _log(f"cfg3 held-out [{s},{e}) {time.time() - t1:.1f} s")
        lab = ds.train_labels
        for p in range(len(ws)):
            errors[p] = int(np.sum(lab[nn[p]] != lab))
        res.update(windows=np.array(ws, np.int64), errors=errors, nn=nn.astype(np.int32))
    else:
        raise ValueError(c)
    res["oracle_seconds"] = np.float64(time.time() - t0)
    res["threads"] = np.int64(threads)
    np.savez_compressed(out + ".tmp.npz", **res)
    os.replace(out + ".tmp.npz", out)
    for f in os.listdir(PARTIAL) if os.path.isdir(PARTIAL) else []:
        if f.startswith(f"cfg{c}_"):
            os.remove(os.path.join(PARTIAL, f))
    _log(f"wrote {out} ({time.time() - t0:.0f} s)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[0, 1, 3, 2, 4])
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--chunk", type=int, default=256)
    a = ap.parse_args()
    oracle.build()
    for c in a.configs:
        golden_cfg(c, a.threads, a.chunk if c != 3 else 64)


if __name__ == "__main__":
    main()
