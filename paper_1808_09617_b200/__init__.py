"""paper_1808_09617_b200 -- exact NN-DTW with the LB_Kim -> LB_Enhanced^V cascade
(arxiv 1808.09617) as hand-written CUDA for B200 (sm_100a) behind a C ABI (include/nndtw.h).

Modules:
  nndtw  -- ctypes binding of libnndtw.so (the only compute path; no CPU fallback)
  dist   -- train-set sharding over ranks with an allreduce-min combine (torch.distributed)
  build  -- nvcc build of libnndtw.so
"""
from . import nndtw  # noqa: F401
from .nndtw import (Model, NNDTWError, Prediction, classify, dtw_batch, envelopes,  # noqa: F401
                    lb_enhanced, loocv_window, series_stats)
