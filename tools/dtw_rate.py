"""Raw DTW kernel rate (no abandoning): nndtw_dtw_batch over P full pairs, CUDA-event timed.

  python tools/dtw_rate.py [L:w:P ...]      default: 512:103:200000 256:26:400000 2048:2047:3000

Prints in-band GCUPS per shape (cells(L,w) = L(2w+1) - w(w+1) per pair) and, with --lb,
the LB tile kernel's pair-column rate on a config-2-shaped slice.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402


def cells(L, w):
    w = min(w, L - 1)
    return L * (2 * w + 1) - w * (w + 1)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    shapes = args or ["512:103:200000", "256:26:400000", "2048:2047:3000"]
    rng = np.random.default_rng(1)
    for s in shapes:
        L, w, P = (int(x) for x in s.split(":"))
        ds = datagen.make_dataset(2 if L == 512 else (4 if L == 2048 else 1), n_train=2048,
                                  n_test=0)
        X = torch.as_tensor(ds.train[:, :L] if ds.train.shape[1] >= L else
                            np.resize(ds.train, (2048, L)).astype(np.float32), device="cuda")
        X = X.contiguous()
        ia = torch.as_tensor(rng.integers(0, 2048, P), dtype=torch.int32, device="cuda")
        if "--ia0" in sys.argv:  # one query row for every pair (shared-A experiments)
            ia.zero_()
        ib = torch.as_tensor(rng.integers(0, 2048, P), dtype=torch.int32, device="cuda")
        ms = timed(lambda: nndtw.dtw_batch(X, X, w, ia, ib))
        g = P * cells(L, w) / (ms * 1e-3) / 1e9
        print(f"dtw L={L} w={w} pairs={P}: {ms:.2f} ms  {g:.0f} GCUPS")
    if "--lb" in sys.argv:
        ds = datagen.make_dataset(2, n_train=100000, n_test=1000)
        t = torch.as_tensor(ds.train, device="cuda")
        q = torch.as_tensor(ds.test, device="cuda")
        U, Lo, kim = nndtw.envelopes(t, 103)
        qk = nndtw.series_stats(q)
        ms = timed(lambda: nndtw.lb_enhanced(q, t, U, Lo, 103, 5, True, qk, kim))
        pc = q.shape[0] * t.shape[0] * (512 - 10)
        print(f"lb 1000x100000 L=512: {ms:.2f} ms  {pc / ms / 1e6:.0f} G pair-cols/s")


if __name__ == "__main__":
    main()
