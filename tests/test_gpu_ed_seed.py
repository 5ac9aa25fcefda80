"""nndtw_ed_seed (ed_seed.cu): the Euclidean-nearest train series of every query, the paper's
candidate order, computed on the tensor cores from the bf16-rounded piecewise-
aggregate approximations (means over f points, f the smallest power of two with ceil(L/f) <= 128).

Checked against the same quantity recomputed here in fp64 from the bf16-rounded PAAs: the chosen
index must attain the minimum up to the fp32 accumulation's rounding (a near-tie may pick either),
and its distance must be the recomputed one within that rounding.  Shapes cover ragged query and
train counts (partial 128-row and 256-row tiles), one and two K-chunks, f = 1 .. 16 (L not a
multiple of f) and more units than SMs."""
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
    f = 1
    while -(-L // f) > 128:
        f *= 2
    Lp = -(-L // f) * f

    def paa(x):
        xp = torch.nn.functional.pad(x, (0, Lp - L))
        return xp.reshape(x.shape[0], -1, f).sum(2) * (1.0 / f)

    qp, tp = paa(q), paa(t)
    qb = qp.to(torch.bfloat16).double()
    tb = tp.to(torch.bfloat16).double()
    qn = (qp.double() ** 2).sum(1)
    tn = (tp.double() ** 2).sum(1)
    ed = (qn[:, None] + tn[None, :] - 2.0 * (qb @ tb.T)).cpu().numpy()
    best = ed.min(axis=1)
    chosen = ed[np.arange(nq), idx]
    scale = (qn.cpu().numpy()[:, None] + tn.cpu().numpy()[None, :]).max(axis=1)
    tol = 2e-4 * scale + 1e-6
    assert np.all(idx >= 0) and np.all(idx < nt)
    assert np.all(chosen <= best + tol), np.nonzero(chosen > best + tol)[0][:8]
    assert np.all(np.abs(dist - np.maximum(chosen, 0.0)) <= tol)


@pytest.mark.parametrize("nq,nt,L", [(1, 1, 8), (5, 300, 64), (128, 256, 128), (129, 257, 100),
                                     (300, 1000, 512), (1000, 5000, 300), (37, 70000, 256),
                                     (50, 900, 2048), (20, 300, 1999)])
def test_ed_seed_argmin(dev, nq, nt, L):
    _check(nq, nt, L)


def test_ed_seed_config2_shape(dev):
    """Config 2's shape (L = 512) at 2000 queries x 100,000 train series (many units per SM)."""
    _check(2000, 100000, 512, seed=3)


def test_ed_seed_rejects_bad_arguments(dev):
    from paper_1808_09617_b200 import nndtw
    lib = nndtw.load()
    assert lib.nndtw_ed_seed(None, -1, None, 0, 8, None, 0, None, None) != 0
    assert lib.nndtw_ed_seed(None, 0, None, 0, 0, None, 0, None, None) != 0
