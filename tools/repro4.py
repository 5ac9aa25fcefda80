import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, datagen
from paper_1808_09617_b200 import nndtw
nndtw.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libnndtw_trace.so"))
L, w, nq, nt = 50, 5, 1, 1
rng = np.random.default_rng(3)
Tr = datagen.random_series(rng, nt, L, "walk"); Q = datagen.random_series(rng, nq, L, "walk")
m = nndtw.Model(torch.as_tensor(Tr, device="cuda"), torch.zeros(nt, dtype=torch.int32, device="cuda"), w, 5)
key, ws, st = nndtw.classify_keys(m, torch.as_tensor(Q, device="cuda"), exact=False, stats=False)
torch.cuda.synchronize()
print(hex(int(key[0])))
