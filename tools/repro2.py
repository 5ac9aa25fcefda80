import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_1808_09617_b200 import nndtw
for (L, w, n) in [(50, 5, 1), (50, 5, 2), (50, 5, 33), (64, 5, 1), (64, 6, 1), (50, 4, 1), (128, 13, 1), (512, 103, 1)]:
    rng = np.random.default_rng(0)
    A = datagen.random_series(rng, n, L, "walk"); B = datagen.random_series(rng, n, L, "walk")
    out = nndtw.dtw_batch(torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda"), w).cpu().numpy()
    ref = np.array([oracle.dtw(A[i], B[i], w) for i in range(n)])
    print(L, w, n, "maxrel", float(np.max(np.abs(out - ref) / ref)), out[:2], ref[:2])
