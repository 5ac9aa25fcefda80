import sys
sys.path.insert(0, '/root/repo')
import torch, datagen
from paper_1808_09617_b200 import nndtw
ds = datagen.make_dataset(3)
x = torch.as_tensor(ds.train, device='cuda'); lab = torch.as_tensor(ds.train_labels, device='cuda')
wins = ds.cfg.windows()
for lo, hi in ((34, 50), (50, 67), (67, 84), (84, 101)):
    ws = wins[lo:hi]
    nndtw.loocv_window(x, lab, ws[:1]); torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); err, _, st = nndtw.loocv_window(x, lab, ws, stats=True); e1.record(); torch.cuda.synchronize()
    print(ws[0], ws[-1], round(e0.elapsed_time(e1),1), 'ms', st['cells'], round(st['ms_dtw'],1))
