import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen, oracle
from paper_1808_09617_b200 import nndtw
for (L, w, nq, nt) in [(50, 5, 1, 1), (50, 5, 1, 2), (50, 5, 2, 3), (50, 5, 40, 40), (512, 103, 1, 1), (128, 13, 1, 1)]:
    rng = np.random.default_rng(3)
    Tr = datagen.random_series(rng, nt, L, "walk"); Q = datagen.random_series(rng, nq, L, "walk")
    m = nndtw.Model(torch.as_tensor(Tr, device="cuda"), torch.zeros(nt, dtype=torch.int32, device="cuda"), w, 5)
    key, ws, st = nndtw.classify_keys(m, torch.as_tensor(Q, device="cuda"), exact=False, stats=True)
    k = key.cpu().numpy().astype(np.uint64)
    d = (k >> np.uint64(32)).astype(np.uint32).view(np.float32)
    ridx, rd = oracle.nn(Q, Tr, w, mode="exhaustive")
    print(L, w, nq, nt, "gpu", d[:3], (k & np.uint64(0xffffffff))[:3], "ref", rd[:3], ridx[:3], st["dtw_calls"], st["survivors"])
