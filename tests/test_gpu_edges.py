"""Edge cases of the boundary on the GPU: empty inputs, the error codes of include/nndtw.h,
and the maximum supported length (L = 8192) against the fp64 oracle."""
import ctypes as C

import numpy as np
import pytest

import datagen

from test_gpu_parity import T, _check_nn, assert_rel, dev  # noqa: F401

pytestmark = pytest.mark.gpu


def test_empty_inputs(dev):
    import torch
    from paper_1808_09617_b200 import nndtw
    L, w = 64, 6
    e = torch.empty((0, L), dtype=torch.float32, device=dev)
    x = T(datagen.random_series(np.random.default_rng(0), 5, L, "walk"), dev)
    U, Lo, kim = nndtw.envelopes(e, w)
    assert U.shape == (0, L) and kim.shape == (0, 4)
    assert nndtw.lb_enhanced(e, x, *nndtw.envelopes(x, w)[:2], w, 5).shape == (0, 5)
    Ux, Lx, kx = nndtw.envelopes(x, w)
    assert nndtw.lb_enhanced(x, e, U, Lo, w, 5).shape == (5, 0)
    assert nndtw.dtw_batch(e, e, w).shape == (0,)
    lab = torch.zeros(5, dtype=torch.int32, device=dev)
    pred = nndtw.classify(nndtw.Model(x, lab, w, 5), e)
    assert pred.idx.shape == (0,)
    # empty train set: no candidate -> index -1, label -1, distance +inf
    pred = nndtw.classify(nndtw.Model(e, torch.zeros(0, dtype=torch.int32, device=dev), w, 5), x)
    assert (pred.idx.cpu().numpy() == -1).all() and (pred.label.cpu().numpy() == -1).all()
    assert np.isinf(pred.dist.cpu().numpy()).all()
    err, nn, _ = nndtw.loocv_window(x, lab, [], v=5)
    assert err.shape == (0,)


def test_error_codes(dev):
    import torch
    from paper_1808_09617_b200 import nndtw
    lib = nndtw.load()
    st = nndtw._stream()
    x = T(datagen.random_series(np.random.default_rng(1), 4, 32, "walk"), dev)
    out = torch.empty(4, dtype=torch.float32, device=dev)
    p = nndtw._ptr
    # L < 2 (Algorithm 1 is not admissible at L = 1, reading C11), L > 8192
    assert lib.nndtw_dtw_batch(p(x), p(x), None, None, 4, 1, 0, None, p(out), st) == 2
    assert lib.nndtw_dtw_batch(p(x), p(x), None, None, 4, 9000, 0, None, p(out), st) == 2
    # negative window, V < 1, null pointers, negative count
    assert lib.nndtw_dtw_batch(p(x), p(x), None, None, 4, 32, -1, None, p(out), st) == 3
    lb = torch.empty((4, 4), dtype=torch.float32, device=dev)
    U, Lo, kim = nndtw.envelopes(x, 3)
    assert lib.nndtw_lb_enhanced(p(x), 4, None, p(x), p(U), p(Lo), None, 4, 32, 3, 0, 0, p(lb),
                                 4, st) == 4
    assert lib.nndtw_lb_enhanced(p(x), 4, None, p(x), None, p(Lo), None, 4, 32, 3, 5, 0, p(lb),
                                 4, st) == 1
    assert lib.nndtw_dtw_batch(None, p(x), None, None, 4, 32, 3, None, p(out), st) == 1
    assert lib.nndtw_dtw_batch(p(x), p(x), None, None, -1, 32, 3, None, p(out), st) == 1
    # workspace too small
    key = torch.empty(4, dtype=torch.int64, device=dev)
    ws = torch.empty(16, dtype=torch.uint8, device=dev)
    rc = lib.nndtw_classify(p(x), 4, p(x), p(U), p(Lo), p(kim), 4, 0, -1, 32, 3, 5, 1, p(ws),
                            ws.numel(), p(key), None, st)
    assert rc == 5
    assert b"workspace" in lib.nndtw_last_error()
    # the Python layer rejects non-finite input before any kernel (NaN is dropped by fminf)
    bad = x.clone()
    bad[1, 3] = float("nan")
    with pytest.raises(nndtw.NNDTWError):
        nndtw.Model(bad, torch.zeros(4, dtype=torch.int32, device=dev), 3, 5)


@pytest.mark.parametrize("w", [0, 13, 1000, 8191])
def test_max_length_dtw(dev, oracle_lib, w):
    from paper_1808_09617_b200 import nndtw
    L = 8192
    rng = np.random.default_rng(w)
    A = datagen.random_series(rng, 2, L, "walk")
    B = datagen.random_series(rng, 2, L, "walk")
    A = (A - A.mean(1, keepdims=True)) / A.std(1, keepdims=True)
    B = (B - B.mean(1, keepdims=True)) / B.std(1, keepdims=True)
    A, B = A.astype(np.float32), B.astype(np.float32)
    out = nndtw.dtw_batch(T(A, dev), T(B, dev), w).cpu().numpy()
    ref = np.array([oracle_lib.dtw(A[i], B[i], w) for i in range(2)])
    assert_rel(out, ref, what=f"L=8192 w={w}")


def test_max_length_classify(dev, oracle_lib):
    from paper_1808_09617_b200 import nndtw
    L, w = 8192, 8191
    rng = np.random.default_rng(8)
    Tr = datagen.random_series(rng, 6, L, "walk")
    Tr[5] = Tr[1]
    Q = np.concatenate([Tr[1:2], datagen.random_series(rng, 1, L, "walk")])
    lab = np.arange(6, dtype=np.int32)
    model = nndtw.Model(T(Tr, dev), T(lab, dev), w, 8)
    pred = nndtw.classify(model, T(Q, dev))
    _check_nn(oracle_lib, Tr, lab, Q, w, pred.idx.cpu().numpy(), pred.label.cpu().numpy(),
              pred.dist.cpu().numpy(), V=8)


def test_graphed_classify_and_loocv(dev, oracle_lib):
    """CUDA-graph replay of classify / LOOCV gives the eager (and the oracle's) answers, replay
    after replay, with new inputs copied into the static buffers."""
    import torch
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(0)
    w = ds.cfg.windows()[0]
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    g = nndtw.GraphedClassifier(model, 50)
    for part in (ds.test[:50], ds.test[50:100], ds.test[:50]):
        pred = g(T(part, dev))
        torch.cuda.synchronize()
        _check_nn(oracle_lib, ds.train, ds.train_labels, part, w, pred.idx.cpu().numpy(),
                  pred.label.cpu().numpy(), pred.dist.cpu().numpy())
    x = T(ds.train[:80], dev)
    lab = T(ds.train_labels[:80], dev)
    wins = [0, 3, 13, 40, 127]
    gl = nndtw.GraphedLoocv(x, lab, wins)
    eager, _, _ = nndtw.loocv_window(x, lab, wins)
    for _ in range(2):
        assert np.array_equal(gl().cpu().numpy(), eager.cpu().numpy())
    ref, _ = oracle_lib.loocv(ds.train[:80], ds.train_labels[:80], wins)
    assert np.array_equal(eager.cpu().numpy(), ref)


def test_classify_query_blocking(dev, oracle_lib):
    """A small workspace budget forces query blocks; the answer is unchanged."""
    from paper_1808_09617_b200 import nndtw
    ds = datagen.make_dataset(0)
    w = ds.cfg.windows()[0]
    model = nndtw.Model(T(ds.train, dev), T(ds.train_labels, dev), w, 5)
    pred = nndtw.classify(model, T(ds.test, dev), stats=True, workspace_budget=400_000)
    assert pred.stats["lb_pairs"] == 100 * 100
    _check_nn(oracle_lib, ds.train, ds.train_labels, ds.test, w, pred.idx.cpu().numpy(),
              pred.label.cpu().numpy(), pred.dist.cpu().numpy())


def test_loocv_degenerate_sizes(dev, oracle_lib):
    """LOOCV with n = 1 (the held-out series is never its own neighbour: index -1, an error,
    reading C17) and n = 2, through the ABI against the oracle, including a constant pair
    (DTW = 0 between the two)."""
    import torch
    from paper_1808_09617_b200 import nndtw
    rng = np.random.default_rng(22)
    wins = [0, 4, 15]
    for X in (datagen.random_series(rng, 2, 16, "walk"), np.ones((2, 16), np.float32)):
        for n, lab in ((1, [3]), (2, [3, 4]), (2, [3, 3])):
            lab = np.array(lab, np.int32)
            err, nn, _ = nndtw.loocv_window(T(X[:n], dev), T(lab, dev), wins, v=5, with_nn=True)
            rerr, rnn = oracle_lib.loocv(X[:n], lab, wins, V=5, mode="pruned")
            assert (err.cpu().numpy() == rerr).all()
            assert (nn.cpu().numpy() == rnn).all()
