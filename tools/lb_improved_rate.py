"""Rate of the O(L) LB_Improved kernel on config-1-shaped pairs (1000 x 1000, L = 256, w = 26):
nndtw.lb_improved (tile kernel LB_Keogh pass + the van Herk projection-envelope pass), CUDA-event
timed.  Used for the ncu capture of k_lb_improved_pass.

  python tools/lb_improved_rate.py [L w nq nt]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402


def main():
    L, w, nq, nt = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (256, 26, 1000, 1000)))
    ds = datagen.make_dataset(1 if L == 256 else 2, n_train=nt, n_test=nq)
    q = torch.as_tensor(ds.test[:, :L], device="cuda").contiguous()
    t = torch.as_tensor(ds.train[:, :L], device="cuda").contiguous()
    U, Lo, _ = nndtw.envelopes(t, w)
    nndtw.lb_improved(q, t, w, t_env=(U, Lo))
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nndtw.lb_improved(q, t, w, t_env=(U, Lo))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    print(f"lb_improved L={L} w={w} {nq}x{nt}: {ms:.3f} ms, {nq * nt / ms / 1e6:.1f} G pairs/s")


if __name__ == "__main__":
    main()
