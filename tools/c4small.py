import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
from paper_1808_09617_b200 import nndtw
ds = datagen.make_dataset(4, n_train=4000, n_test=200)
m = nndtw.Model(torch.as_tensor(ds.train, device="cuda"), torch.as_tensor(ds.train_labels, device="cuda"), 2047, 8)
for _ in range(2):
    p = nndtw.classify(m, torch.as_tensor(ds.test, device="cuda"), stats=True)
torch.cuda.synchronize(); print(p.stats)
