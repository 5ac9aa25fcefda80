"""S6 -- train-set sharding over ranks (one process per GPU) with MIN-allreduce combines.

The train set is split into contiguous index ranges, queries are replicated, and every rank
runs S1-S5 on its shard (nndtw_classify without the EXACT flag) in two phases: the seed phase
(S2 bound, S3 seed DTW of each query's argmin-bound candidate) ends with an int64 MIN
all-reduce of the seed keys, so that every shard prunes and abandons against the best seed of
ALL shards (a valid upper bound on the global NN distance) instead of its own -- without it
each shard's survivors grow as the shard shrinks.  Three more MIN all-reduces then give the
exact answer:

1. key   = (fp32 distance bits << 32) | global index  -> global fp32 best (reading C13);
2. f64   = fp64 bits of each rank's near-tie candidates within the global fp32 best's band
           (reading C16) -> global fp64 minimum;
3. out   = (global index << 32) | fp32 bits of candidates whose fp64 value equals it
           -> lowest index among exact fp64 ties.

All keys are < 2^63 (non-negative floats, indices < 2^31, "none" = INT64_MAX), so a signed
int64 MIN is the unsigned MIN.  Messages are Q x 8 bytes per step.  Optionally (split=True)
the search runs in two halves (the survivors of the lowest-bound buckets first, then the rest)
with one more key MIN between them, so that every shard's second half prunes and abandons
against the best distances all shards found in their first half: at 8 shards 4 % fewer DTW
cells, but the extra synchronisation point leaves the projected step time within 1 %
(profiles/round1l_shard_sim.md), so it is off by default.

The per-shard operations are injected (`ShardOps`) so that the combine protocol itself is
tested on CPU with the gloo backend (tests/test_dist_gloo.py); `GpuShardOps` is the product
path through the C ABI.

S8 (LOOCV window search) shards the other way: every rank holds all n series
(each is a candidate for every held-out query), the held-out queries are split into contiguous
ranges, and the per-window error counts are summed with one int64 SUM all-reduce of nw
entries; the best window is then the same on every rank.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import nndtw


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n train series for `rank` of `world`."""
    return (n * rank) // world, (n * (rank + 1)) // world


class ShardOps:
    """Interface of the per-shard steps (all tensors int64 [nq] on the rank's device)."""

    def local_keys(self, q):
        raise NotImplementedError

    # optional two-phase form of local_keys (seed keys, MIN over ranks, then the search)
    seed_keys = None
    search_keys = None
    # optional split search (the lowest-bound survivors, MIN over ranks, then the rest)
    search_a_keys = None
    search_b_keys = None

    def refine(self, q, gkey):
        raise NotImplementedError

    def resolve(self, q, gkey, gf64):
        raise NotImplementedError


class GpuShardOps(ShardOps):
    def __init__(self, model: nndtw.Model, stats: bool = False, stream=None, split: bool = False):
        self.model = model
        self.stats = stats
        self.stream = stream
        self.ws = None
        self.last_stats = None
        if not split:  # one search phase (no mid-search exchange)
            self.search_a_keys = None
            self.search_b_keys = None

    def local_keys(self, q):
        key, ws, st = nndtw.classify_keys(self.model, q, exact=False, stats=self.stats,
                                          stream=self.stream)
        self.ws = ws
        self.last_stats = st
        return key

    def seed_keys(self, q):
        key, ws, st = nndtw.classify_keys(self.model, q, exact=False, stats=self.stats,
                                          stream=self.stream, phase="seed")
        self.ws = ws
        self.last_stats = st
        return key

    def search_keys(self, q, gseed):
        key, _, st = nndtw.classify_keys(self.model, q, exact=False, stats=self.stats,
                                         stream=self.stream, phase="search", key=gseed,
                                         ws=self.ws)
        self.last_stats = nndtw.merge_stats(self.last_stats, st)
        return key

    def search_a_keys(self, q, gseed):
        key, _, st = nndtw.classify_keys(self.model, q, exact=False, stats=self.stats,
                                         stream=self.stream, phase="search_a", key=gseed,
                                         ws=self.ws)
        self.last_stats = nndtw.merge_stats(self.last_stats, st)
        return key

    def search_b_keys(self, q, gkey):
        key, _, st = nndtw.classify_keys(self.model, q, exact=False, stats=self.stats,
                                         stream=self.stream, phase="search_b", key=gkey,
                                         ws=self.ws)
        self.last_stats = nndtw.merge_stats(self.last_stats, st)
        return key

    def refine(self, q, gkey):
        return nndtw.classify_refine(self.model, q, self.ws, gkey, self.stream)

    def resolve(self, q, gkey, gf64):
        return nndtw.classify_resolve(self.model, q, self.ws, gkey, gf64, self.stream)


def combine(ops: ShardOps, q, group=None):
    """Run the 3-step exact combine; returns the final key tensor in key format 1
    ((global index << 32) | fp32 distance bits)."""
    if getattr(ops, "seed_keys", None) is not None:
        key = ops.seed_keys(q)
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)  # global seed best-so-far
        if getattr(ops, "search_a_keys", None) is not None:
            key = ops.search_a_keys(q, key)  # the lowest-bound survivors
            dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)  # global best so far
            key = ops.search_b_keys(q, key)  # the rest, pruned by all shards' best
        else:
            key = ops.search_keys(q, key)
    else:
        key = ops.local_keys(q)
    dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    f64 = ops.refine(q, key)
    dist.all_reduce(f64, op=dist.ReduceOp.MIN, group=group)
    out = ops.resolve(q, key, f64)
    dist.all_reduce(out, op=dist.ReduceOp.MIN, group=group)
    return out


def classify_sharded(model: nndtw.Model, q: torch.Tensor, labels_global: torch.Tensor,
                     group=None, stats: bool = False, stream=None,
                     split: bool = False) -> nndtw.Prediction:
    """Exact 1-NN of every query against the union of all ranks' shards.  `model` holds this
    rank's shard with index_base = its first global index; labels_global is replicated.
    split: exchange the best-so-far once more in the middle of the survivor round."""
    ops = GpuShardOps(model, stats=stats, stream=stream, split=split)
    out = combine(ops, q, group)
    idx, lab, d = nndtw.finalize(out, labels_global, key_format=1, stream=stream)
    return nndtw.Prediction(idx, lab, d, ops.last_stats)


def best_window(errors, windows) -> int:
    """argmin of the error counts, ties to the smallest w (reading C17)."""
    e = [int(x) for x in errors]
    return min(range(len(e)), key=lambda p: (e[p], int(windows[p]))) if e else -1


def loocv_sharded(x: torch.Tensor, labels: torch.Tensor, windows, v: int = 5, group=None,
                  stream=None, shard_fn=None):
    """S8 over ranks: LOOCV error counts for every window in `windows` (absolute w), the
    held-out queries split by shard_range over the ranks of `group`, all n series replicated
    (self excluded by the kernel).  Returns (errors int64 [nw] on every rank, best window index).

    shard_fn(q_begin, q_end) -> int64 [nw] computes one shard's counts; the default is the C-ABI
    path (nndtw.loocv_window); the gloo tests inject the oracle."""
    n = x.shape[0]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(n, rank, world)
    if shard_fn is None:
        def shard_fn(a, b):
            return nndtw.loocv_window(x, labels, windows, v=v, q_begin=a, q_end=b,
                                      stream=stream)[0]
    errors = shard_fn(lo, hi).to(torch.int64)
    dist.all_reduce(errors, op=dist.ReduceOp.SUM, group=group)
    return errors, best_window(errors.cpu().tolist(), windows)
