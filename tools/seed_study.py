"""How close do the k lowest-bound candidates' DTWs come to each query's final NN distance?

For config 2 queries (a subset): the full cascade bound for all pairs (nndtw_lb_enhanced with
LB_Kim), the k lowest-bound candidates per query DTW'd exactly (nndtw_dtw_batch), and the
best-so-far they give against the final answer (nndtw.classify).  Tells what extra seed rounds
before the survivor round could buy (the survivor round with the final best-so-far preset is
2.8 % faster, tools/threshold_gap.py).

  python tools/seed_study.py [--queries 1000]
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
    ap.add_argument("--queries", type=int, default=1000)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    ds = datagen.make_dataset(2)
    w, V = ds.cfg.windows()[0], 5
    t = torch.as_tensor(ds.train, device=dev)
    q = torch.as_tensor(ds.test[:a.queries], device=dev)
    model = nndtw.Model(t, torch.as_tensor(ds.train_labels, device=dev), w, V)
    final = nndtw.classify(model, q).dist.double()
    U, Lo, kim = nndtw.envelopes(t, w)
    lb = nndtw.lb_enhanced(q, t, U, Lo, w, V, True, None, kim)
    nq = q.shape[0]
    order = torch.argsort(lb, dim=1)[:, :16]
    ia = torch.arange(nq, device=dev, dtype=torch.int32).repeat_interleave(16)
    ib = order.reshape(-1).to(torch.int32)
    d = nndtw.dtw_batch(q, t, w, ia, ib).double().reshape(nq, 16)
    # the two-stage S2's list size against its threshold: pairs with partial value
    # P = max(LB_Kim, boundary + bands) <= c * final (stage B computes the bridge for these)
    part = nndtw.lb_enhanced(q, t, U, Lo, w, V, True, None, kim, partial=True)
    fin = final.float().unsqueeze(1)
    for c in (1.0, 1.1, 1.2, 1.3, 1.5):
        frac = (part <= fin * c).double().mean().item()
        print(f"pairs with P <= {c:.1f} x final: {frac * 100:5.2f} %")
    p1 = part.argmin(dim=1).to(torch.int32)
    d1 = nndtw.dtw_batch(q, t, w, torch.arange(nq, device=dev, dtype=torch.int32), p1).double()
    print(f"partial-argmin seed: mean bsf / final = {(d1 / final.clamp_min(1e-30)).mean().item():.3f}, "
          f"listed at its bsf: {(part <= d1.float().unsqueeze(1)).double().mean().item() * 100:.2f} %")
    # top-k partial-value candidates, and the paper's Euclidean order: the ED argmin
    # (|q|^2 + |t|^2 - 2 q.t, here a torch matmul -- a seed choice only, its DTW is exact)
    po = torch.argsort(part, dim=1)[:, :8]
    dp = nndtw.dtw_batch(q, t, w, torch.arange(nq, device=dev, dtype=torch.int32)
                         .repeat_interleave(8), po.reshape(-1).to(torch.int32)).double()
    dp = dp.reshape(nq, 8)
    for k in (1, 2, 4, 8):
        print(f"top-{k} partial-value candidates: mean bsf / final = "
              f"{(dp[:, :k].min(dim=1).values / final.clamp_min(1e-30)).mean().item():.3f}")
    ed = (q * q).sum(1, keepdim=True) + (t * t).sum(1).unsqueeze(0) - 2.0 * (q @ t.T)
    e1 = ed.argmin(dim=1).to(torch.int32)
    de = nndtw.dtw_batch(q, t, w, torch.arange(nq, device=dev, dtype=torch.int32), e1).double()
    print(f"ED-argmin seed: NN found for {(de <= final * (1 + 1e-6)).double().mean().item() * 100:.1f} % "
          f"of queries, mean bsf / final = {(de / final.clamp_min(1e-30)).mean().item():.3f}, "
          f"listed at its bsf: {(part <= de.float().unsqueeze(1)).double().mean().item() * 100:.2f} %")
    for f in (2, 4):  # the same on series averaged over f consecutive points (PAA)
        qp = q.reshape(nq, -1, f).mean(2)
        tp = t.reshape(t.shape[0], -1, f).mean(2)
        edp = (qp * qp).sum(1, keepdim=True) + (tp * tp).sum(1).unsqueeze(0) - 2.0 * (qp @ tp.T)
        ep = edp.argmin(dim=1).to(torch.int32)
        if f == 4:  # the k Euclidean-nearest (PAA) candidates as seeds
            eo = torch.argsort(edp, dim=1)[:, :8]
            de8 = nndtw.dtw_batch(q, t, w, torch.arange(nq, device=dev, dtype=torch.int32)
                                  .repeat_interleave(8), eo.reshape(-1).to(torch.int32)).double()
            de8 = de8.reshape(nq, 8)
            for k in (1, 2, 4, 8):
                bk = de8[:, :k].min(dim=1).values
                print(f"top-{k} ED (PAA/4) candidates: mean bsf / final = "
                      f"{(bk / final.clamp_min(1e-30)).mean().item():.3f}, listed at its bsf: "
                      f"{(part <= bk.float().unsqueeze(1)).double().mean().item() * 100:.2f} %")
        del edp
        dpa = nndtw.dtw_batch(q, t, w, torch.arange(nq, device=dev, dtype=torch.int32), ep).double()
        print(f"ED argmin on PAA/{f}: mean bsf / final = "
              f"{(dpa / final.clamp_min(1e-30)).mean().item():.3f}, listed at its bsf: "
              f"{(part <= dpa.float().unsqueeze(1)).double().mean().item() * 100:.2f} %")
    for k in (1, 2, 4, 8, 16):
        best = d[:, :k].min(dim=1).values
        hit = (best <= final * (1 + 1e-6)).double().mean().item()
        ratio = (best / final.clamp_min(1e-30)).mean().item()
        print(f"top-{k:2d} full-bound candidates: NN found for {hit * 100:5.1f} % of queries, "
              f"mean bsf / final = {ratio:.3f}")


if __name__ == "__main__":
    main()
