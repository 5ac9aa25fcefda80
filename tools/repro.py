"""Small reproduction driver for debugging one DTW / classify shape on the GPU."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen
from paper_1808_09617_b200 import nndtw

L, w, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "batch"
rng = np.random.default_rng(0)
A = torch.as_tensor(datagen.random_series(rng, n, L, "walk"), device="cuda")
B = torch.as_tensor(datagen.random_series(rng, n, L, "walk"), device="cuda")
if mode == "batch":
    out = nndtw.dtw_batch(A, B, w)
    torch.cuda.synchronize()
    print("ok", out[:4].tolist())
else:
    m = nndtw.Model(B, torch.zeros(n, dtype=torch.int32, device="cuda"), w, 1)
    p = nndtw.classify(m, A, stats=True)
    torch.cuda.synchronize()
    print("ok", p.idx[:4].tolist(), p.stats)
