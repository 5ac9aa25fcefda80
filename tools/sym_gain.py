"""How much DTW work does the symmetric bound remove on config 2? (classify with
max(LB(q,t), LB(t,q)) for all pairs vs the one-sided bound; stage times and counters)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
ds = datagen.make_dataset(2, n_test=nq)
tr = torch.as_tensor(ds.train, device="cuda")
lab = torch.as_tensor(ds.train_labels, device="cuda")
q = torch.as_tensor(ds.test, device="cuda")
for sym in (False, True, False, True):
    m = nndtw.Model(tr, lab, 103, 5, check=False, symmetric=sym)
    p = nndtw.classify(m, q, stats=True, check=False)
    st = p.stats
    print(f"symmetric={sym}: lb {st['ms_lb']:.1f} ms  dtw {st['ms_dtw']:.1f} ms  other "
          f"{st['ms_other']:.1f} ms  survivors {st['survivors']}  calls {st['dtw_calls']}  "
          f"cells {st['cells']:.4g}")
