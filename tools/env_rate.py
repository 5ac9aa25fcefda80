"""S1 envelope kernel rate: nndtw_envelopes on a config-shaped train set, CUDA-event timed.

  python tools/env_rate.py [N L w reps]     default: config 2 (100000 x 512, w=103)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1808_09617_b200 import nndtw  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
L = int(sys.argv[2]) if len(sys.argv) > 2 else 512
w = int(sys.argv[3]) if len(sys.argv) > 3 else 103
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
x = torch.randn(N, L, device="cuda").cumsum(1).contiguous()
U = torch.empty_like(x)
Lo = torch.empty_like(x)
kim = torch.empty((N, 4), dtype=torch.int32, device=x.device)
lib = nndtw.load()
st = nndtw._stream(None)
P = nndtw._ptr


def launch():
    assert lib.nndtw_envelopes(P(x), N, L, w, P(U), P(Lo), P(kim), st) == 0


launch()
torch.cuda.synchronize()
ts = []
for _ in range(5):  # back-to-back launches between one event pair: no host gaps in the timing
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / reps)
ms = float(np.median(ts))
print(f"envelopes N={N} L={L} w={w}: {ms:.4f} ms  {N * L * 12 / ms / 1e6:.0f} GB/s (12 B/elt)")
