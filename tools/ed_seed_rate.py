import sys, torch
sys.path.insert(0, '/root/repo')
import datagen
from paper_1808_09617_b200 import nndtw
ds = datagen.make_dataset(2)
q = torch.as_tensor(ds.test, device='cuda'); t = torch.as_tensor(ds.train, device='cuda')
nndtw.ed_seed(q, t); torch.cuda.synchronize()
for r in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); idx, d = nndtw.ed_seed(q, t); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"ed_seed 10000 x 100000 x 512: {ms:.3f} ms  {2*1e4*1e5*512/ms/1e9:.0f} TFLOP/s")
