"""The N>1 path on CPU: world_size-2 gloo process groups run the real combine protocol of
paper_1808_09617_b200.dist (three int64 MIN all-reduces) with shard operations emulated from
the oracle (the GPU kernels are not available here).  The emulation reproduces what the
kernels hand to the collectives: fp32 distances rounded from fp64, global indices, the fp64
near-tie re-rank; the test checks the combined answer is the oracle's global 1-NN."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen

NONE64 = 0x7FFFFFFFFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShardOps:
    """CPU emulation of GpuShardOps on one shard (test infrastructure: uses the oracle)."""

    def __init__(self, T, lo, hi, w, f32_jitter=None):
        import oracle
        self.o = oracle
        self.T, self.lo, self.hi, self.w = T, lo, hi, w
        self.f32_jitter = f32_jitter
        self.cand = {}

    def _d64(self, q, n):
        return self.o.dtw(q, self.T[n], self.w)

    def local_keys(self, Q):
        keys = []
        self.d32 = {}
        for i, q in enumerate(Q.numpy()):
            best = NONE64
            for n in range(self.lo, self.hi):
                d = np.float32(self._d64(q, n))
                if self.f32_jitter is not None:  # model fp32 rounding noise of the kernels
                    d = np.float32(d * (1 + self.f32_jitter[i, n]))
                self.d32[(i, n)] = d
                k = (int(np.float32(d).view(np.uint32)) << 32) | n
                best = min(best, k)
            keys.append(best)
        return torch.tensor(keys, dtype=torch.int64)

    def refine(self, Q, gkey):
        L = Q.shape[1]
        eps_t = (4 * L + 8) * 2.0 ** -24
        out = []
        self.band = {}
        for i, q in enumerate(Q.numpy()):
            gb = np.uint32(int(gkey[i]) >> 32).view(np.float32)
            best = NONE64
            for n in range(self.lo, self.hi):
                if self.d32[(i, n)] <= gb * np.float32(1 + eps_t):
                    d64 = self._d64(q, n)
                    self.band[(i, n)] = d64
                    best = min(best, int(np.float64(d64).view(np.int64)))
            out.append(best)
        return torch.tensor(out, dtype=torch.int64)

    def resolve(self, Q, gkey, gf64):
        out = []
        for i in range(Q.shape[0]):
            best = NONE64
            for (qi, n), d64 in self.band.items():
                if qi == i and int(np.float64(d64).view(np.int64)) == int(gf64[i]):
                    best = min(best, (n << 32) | int(self.d32[(i, n)].view(np.uint32)))
            out.append(best)
        return torch.tensor(out, dtype=torch.int64)


class OracleTwoPhaseShardOps(OracleShardOps):
    """The two-phase form (GpuShardOps.seed_keys / search_keys): the seed key of each query is
    the shard's argmin-bound candidate (LB_Kim -> LB_Enhanced cascade, oracle); the search
    starts from the MIN over ranks of the seed keys -- possibly another rank's candidate, which
    this rank's refine/resolve never see -- and keeps the smaller of it and the local best."""

    def seed_keys(self, Q):
        U, Lo = self.o.envelopes(self.T[self.lo:self.hi], self.w)
        keys = []
        for q in Q.numpy():
            lbs = [self.o.lb_cascade(q, self.T[n], U[n - self.lo], Lo[n - self.lo], self.w, 5)
                   for n in range(self.lo, self.hi)]
            n = self.lo + int(np.argmin(lbs))
            d = np.float32(self._d64(q, n))
            keys.append((int(d.view(np.uint32)) << 32) | n)
        return torch.tensor(keys, dtype=torch.int64)

    def search_keys(self, Q, gseed):
        local = self.local_keys(Q)
        return torch.minimum(local, gseed)


class OracleSplitShardOps(OracleTwoPhaseShardOps):
    """The split search (GpuShardOps.search_a_keys / search_b_keys): the first half searches the
    shard's candidates with the lowest bounds (here: the first half of its index range) from the
    global seed, the keys are MIN-combined again, and the second half continues from that."""

    def search_a_keys(self, Q, gseed):
        local = self.local_keys(Q)  # (emulation: the full local search; the halves only order it)
        return torch.minimum(local, gseed)

    def search_b_keys(self, Q, gkey):
        return torch.minimum(self.local_keys(Q), gkey)


def _worker(rank, world, port, T, Q, w, jitter, ret, two_phase=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1808_09617_b200.dist import combine, shard_range
    lo, hi = shard_range(T.shape[0], rank, world)
    cls = {False: OracleShardOps, True: OracleTwoPhaseShardOps,
           "split": OracleSplitShardOps}[two_phase]
    ops = cls(T, lo, hi, w, jitter)
    out = combine(ops, torch.as_tensor(Q))
    ret[rank] = [int(x) >> 32 for x in out]
    dist.destroy_process_group()


@pytest.mark.parametrize("world,two_phase", [(2, False), (3, False), (2, True), (3, True),
                                              (2, "split"), (3, "split")])
def test_sharded_combine_matches_global_nn(oracle_lib, world, two_phase):
    rng = np.random.default_rng(world)
    L, w = 10, 2
    T = datagen.random_series(rng, 23, L, "int")
    T[15] = T[4]      # exact duplicate in another shard: lowest global index must win
    T[20] = T[2]
    Q = datagen.random_series(rng, 9, L, "int")
    Q[0] = T[15]
    # fp32 noise that may reorder near-ties -- the fp64 re-rank must undo it
    jitter = rng.uniform(-3e-7, 3e-7, size=(9, 23))
    mgr = mp.Manager()
    ret = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, T, Q, w, jitter, ret, two_phase), nprocs=world,
             join=True)
    ridx, _ = oracle_lib.nn(Q, T, w, mode="exhaustive")
    for r in range(world):
        assert list(ret[r]) == list(ridx), (r, ret[r], ridx)


def test_shard_range_partition():
    from paper_1808_09617_b200.dist import shard_range
    for n in (1, 7, 100000):
        for world in (1, 2, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def _loocv_worker(rank, world, port, X, lab, windows, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1808_09617_b200.dist import loocv_sharded

    def shard_fn(a, b):  # one rank's held-out range, emulated with the oracle
        return torch.as_tensor(oracle.loocv(X, lab, windows, V=2, q_begin=a, q_end=b,
                                            threads=1)[0])
    errors, best = loocv_sharded(torch.as_tensor(X), torch.as_tensor(lab), windows,
                                 shard_fn=shard_fn)
    ret[rank] = (errors.tolist(), best)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_loocv_sharded_sums_to_global(oracle_lib, world):
    """S8 sharded over held-out queries: the SUM all-reduce of per-shard counts equals the
    unsharded LOOCV, and every rank agrees on the best window (ties to the smallest w)."""
    from paper_1808_09617_b200.dist import best_window
    rng = np.random.default_rng(40 + world)
    X = datagen.random_series(rng, 17, 12, "walk")
    lab = (np.arange(17) % 3).astype(np.int32)
    windows = [0, 1, 2, 4, 11]
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_loocv_worker, args=(world, _free_port(), X, lab, windows, ret), nprocs=world,
             join=True)
    ref, _ = oracle_lib.loocv(X, lab, windows, V=2, mode="exhaustive")
    for r in range(world):
        assert ret[r][0] == list(ref), (r, ret[r], ref)
        assert ret[r][1] == best_window(ref, windows)


def test_best_window_ties_to_smallest_w():
    from paper_1808_09617_b200.dist import best_window
    assert best_window([3, 1, 1, 2], [0, 5, 9, 12]) == 1
    assert best_window([2, 2], [7, 3]) == 1
    assert best_window([], []) == -1
