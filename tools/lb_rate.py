"""LB tile kernel rate on a config-2-shaped slice (Q=1000 x N=100000, L=512, w=103, V=5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ds = datagen.make_dataset(2, n_train=100000, n_test=nq)
t = torch.as_tensor(ds.train, device="cuda")
q = torch.as_tensor(ds.test, device="cuda")
U, Lo, kim = nndtw.envelopes(t, 103)
qk = nndtw.series_stats(q)
ts = []
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    nndtw.lb_enhanced(q, t, U, Lo, 103, 5, True, qk, kim)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"lb {nq}x100000 L=512: {ms:.2f} ms  {nq * 100000 * 502 / ms / 1e6:.0f} G pair-cols/s")
