"""How much DTW work the live best-so-far costs over an oracle threshold (config 2).

Runs the classify search twice on the same queries: once as the product does (seed rounds,
then the survivors in LB-bucket order against the live per-query best-so-far), once with every
query's best-so-far preset to its final answer before the survivor round (what a perfect
survivor order would reach).  The gap in DTW calls / cells / ms bounds what any reordering of
the survivors could still save.

  python tools/threshold_gap.py [--queries 10000]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_1808_09617_b200 import nndtw  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=10000)
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    ds = datagen.make_dataset(a.config)
    w = ds.cfg.windows()[0]
    model = nndtw.Model(torch.as_tensor(ds.train, device=dev),
                        torch.as_tensor(ds.train_labels, device=dev), w, 5)
    q = torch.as_tensor(ds.test[:a.queries], device=dev)
    for rep in range(2):
        key, ws, s0 = nndtw.classify_keys(model, q, exact=False, phase="seed", stats=True)
        key, ws, s1 = nndtw.classify_keys(model, q, exact=False, phase="search", key=key, ws=ws,
                                          stats=True)
    final = key.clone()
    st = nndtw.merge_stats(s0, s1)
    print(f"live best-so-far : dtw_calls {st['dtw_calls']:>11,} cells {st['cells']:.4e} "
          f"ms_dtw {s1['ms_dtw']:.1f} survivors {st['survivors']:,}")
    # an extra seed from the paper's Euclidean order: the ED argmin's exact DTW,
    # folded into the seed keys before the survivor round (the lists are already built)
    t = model.t
    ed = (q * q).sum(1, keepdim=True) + (t * t).sum(1).unsqueeze(0) - 2.0 * (q @ t.T)
    e1 = ed.argmin(dim=1).to(torch.int32)
    del ed
    de = nndtw.dtw_batch(q, t, model.w, torch.arange(q.shape[0], device=dev,
                                                      dtype=torch.int32), e1)
    ked = (de.view(torch.int32).to(torch.int64) << 32) | e1.to(torch.int64)
    for rep in range(2):
        key, ws, s0 = nndtw.classify_keys(model, q, exact=False, phase="seed", stats=True)
        key = torch.minimum(key, ked)
        key, ws, s1 = nndtw.classify_keys(model, q, exact=False, phase="search", key=key, ws=ws,
                                          stats=True)
    st = nndtw.merge_stats(s0, s1)
    assert torch.equal(key, final)
    print(f"+ ED-argmin seed : dtw_calls {st['dtw_calls']:>11,} cells {st['cells']:.4e} "
          f"ms_dtw {s1['ms_dtw']:.1f} survivors {st['survivors']:,}")
    key, ws, s0 = nndtw.classify_keys(model, q, exact=False, phase="seed", stats=True)
    key = torch.minimum(key, final)
    key, ws, s1 = nndtw.classify_keys(model, q, exact=False, phase="search", key=key, ws=ws,
                                      stats=True)
    st = nndtw.merge_stats(s0, s1)
    assert torch.equal(key, final)
    print(f"final (oracle)   : dtw_calls {st['dtw_calls']:>11,} cells {st['cells']:.4e} "
          f"ms_dtw {s1['ms_dtw']:.1f} survivors {st['survivors']:,}")


if __name__ == "__main__":
    main()
