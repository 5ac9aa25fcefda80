import sys, os, json
sys.path.insert(0, '/root/repo')
import torch, numpy as np, datagen
from paper_1808_09617_b200 import nndtw
ds = datagen.make_dataset(3)
x = torch.as_tensor(ds.train, device='cuda'); lab = torch.as_tensor(ds.train_labels, device='cuda')
wins = ds.cfg.windows()
nndtw.loocv_window(x, lab, wins[:3])
torch.cuda.synchronize()
for chunk in (wins[:10], wins[10:40], wins[40:70], wins[70:]):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); err, _, st = nndtw.loocv_window(x, lab, chunk, stats=True); e1.record(); torch.cuda.synchronize()
    print(chunk[0], chunk[-1], round(e0.elapsed_time(e1),1), {k: (round(v,2) if isinstance(v,float) else v) for k,v in st.items()})
# without stats: no per-window host synchronisation
for rep in range(2):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); err, _, _ = nndtw.loocv_window(x, lab, wins); e1.record(); torch.cuda.synchronize()
    print('all 101 windows, no stats:', round(e0.elapsed_time(e1), 1), 'ms')
