"""nndtw_ed_seed (ed_seed.cu): the Euclidean-nearest train series of every query, the paper's
candidate order, computed on the tensor cores from bf16-rounded series.

Checked against the same quantity recomputed here in fp64 from the bf16-rounded inputs: the
chosen index must attain the minimum up to the fp32 accumulation's rounding (a near-tie may pick
either), and its distance must be the recomputed one within that rounding.  Shapes cover ragged
query and train counts (partial 128-row and 256-row tiles), every K-chunk count (L up to 512,
L not a multiple of 64) and more units than SMs."""
import numpy as np
import pytest
import torch

import datagen

from test_gpu_parity import dev  # noqa: F401

pytestmark = pytest.mark.gpu


def _check(nq, nt, L, kind="walk", seed=0):
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(seed + nq * 7 + nt + L)
    Q = datagen.random_series(rng, nq, L, kind)
    Tn = datagen.random_series(rng, nt, L, kind)
    Tn[min(3, nt - 1)] = Q[0]
    dev = torch.device("cuda:0")
    q = torch.as_tensor(Q, device=dev)
    t = torch.as_tensor(Tn, device=dev)
    idx, dist = nndtw.ed_seed(q, t)
    idx = idx.cpu().numpy()
    dist = dist.cpu().numpy()
    qb = q.to(torch.bfloat16).double()
    tb = t.to(torch.bfloat16).double()
    qn = (q.double() ** 2).sum(1)
    tn = (t.double() ** 2).sum(1)
    ed = (qn[:, None] + tn[None, :] - 2.0 * (qb @ tb.T)).cpu().numpy()
    best = ed.min(axis=1)
    chosen = ed[np.arange(nq), idx]
    scale = (qn.cpu().numpy()[:, None] + tn.cpu().numpy()[None, :]).max(axis=1)
    tol = 2e-4 * scale + 1e-6
    assert np.all(idx >= 0) and np.all(idx < nt)
    assert np.all(chosen <= best + tol), np.nonzero(chosen > best + tol)[0][:8]
    assert np.all(np.abs(dist - np.maximum(chosen, 0.0)) <= tol)


@pytest.mark.parametrize("nq,nt,L", [(1, 1, 8), (5, 300, 64), (128, 256, 128), (129, 257, 100),
                                     (300, 1000, 512), (1000, 5000, 300), (37, 70000, 256)])
def test_ed_seed_argmin(dev, nq, nt, L):
    _check(nq, nt, L)


def test_ed_seed_config2_shape(dev):
    """Config 2's shape (L = 512) at 2000 queries x 100,000 train series (many units per SM)."""
    _check(2000, 100000, 512, seed=3)


def test_ed_seed_rejects_long_rows(dev):
    from paper_1808_09617_b200 import nndtw
    q = torch.zeros((4, 513), device="cuda:0")
    with pytest.raises(nndtw.NNDTWError):
        nndtw.ed_seed(q, q)
