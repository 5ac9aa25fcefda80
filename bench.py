"""Benchmark: NN-DTW queries/s with the LB_Kim -> LB_Enhanced^V cascade (BASELINE.json metric).

Workload (default): BASELINE.json configs[2] "Large search" -- N=100,000 train, Q=10,000
queries, L=512, W=0.2*L (w=103), V=5, 20 classes -- the config whose train set is sharded over
GPUs.  One step = the whole hot path S1-S7: train envelopes + Kim features
(S1), the cascade bound of all Q x N pairs (S2), seed / prune / compaction (S3), DTW with early
abandoning (S4), argmin + fp64 near-tie re-rank (S5, S7) and, for N>1 GPUs, the MIN
all-reduce shard combine (S6).  Inputs are resident in HBM when the timed region starts; the
working set (4 GB LB matrix, 600 MB series + envelopes) is larger than the 126 MB L2.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import datagen  # noqa: E402

METRIC = "NN-DTW queries/s (LB_Enhanced^V cascade) at 1/2/4/8 B200; DTW GCUPS"
# L2 -> SM read rate for whole 2 KB rows at 16 warps/SM (tools/l2_roof.cu, measured on B200)
L2_ROW_GBS = 18301.0


def envelope_kernel(L: int, w: int) -> str:
    """Which S1 kernel launch_envelopes (envelopes.cu) picks: the direct form for w >= 16 when
    its padded shared-memory arrays fit, van Herk otherwise (same rule as the launcher)."""
    w = min(w, L - 1)
    if L <= 256 or w < 16:
        return "k_envelopes"
    tps = 32 * ((L + 511) // 512)
    if tps > 256:
        return "k_envelopes"
    groups = max(64, tps) // tps
    q = w >> 4
    plen = (17 * (2 * (q + 1) + tps) + 1) & ~1
    zlen = tps + 2 * (q + 1)
    zall = (3 * zlen + 1) & ~1
    smem = groups * ((2 * plen + zall) * 8 + 16 * 16 + 2 * 16 * tps * 4)
    return "k_env_direct" if smem <= 112 * 1024 else "k_envelopes"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def dtw_cell_peak_gcups(num_sms: int, sm_mhz: float) -> float:
    """Pipe roof of the DTW recurrence: every DP cell needs one 3-way min.
    FMNMX3 issues at half rate (tools/pipebench.cu on B200: 0.495 warp-instr/clk/SMSP, i.e.
    16 lanes/clk), and the arithmetic (a-b, then (a-b)^2 + min) costs the FMA pipe the same 2
    cycles per 32 cells; so each SM retires at most 4 x 16 = 64 cells per clock."""
    return num_sms * 64.0 * sm_mhz * 1e6 / 1e9


def lb_pair_col_peak(num_sms: int, sm_mhz: float) -> float:
    """Pipe roof of the LB_Keogh bridge: per (pair, column) two subtractions and
    one FFMA on the FMA pipe (32 lanes/clk/SMSP; packed FADD2 issues at half rate, so packing
    saves issue slots, not pipe cycles) -> 4 x 32 / 3 = 42.7 pair-columns per SM per clock."""
    return num_sms * 128.0 / 3.0 * sm_mhz * 1e6 / 1e9


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each hot kernel, from the
    committed `ncu --set full` capture of this command (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_baseline_oracle(ds, w, V, target_s=15.0):
    """The fp64 oracle's paper-pruned search (mode ii: ED order, Algorithm 1, DTW with
    abandoning), as it stands, on a bounded query sample, all host cores."""
    import oracle
    oracle.build()
    cores = oracle.default_threads()
    U, Lo = oracle.envelopes(ds.train, w)
    n = cores
    t0 = time.perf_counter()
    oracle.nn(ds.test[:n], ds.train, w, V=V, mode="pruned", envelopes_UL=(U, Lo))
    el = time.perf_counter() - t0
    # scale the sample to about target_s seconds (bounded)
    n2 = int(min(ds.test.shape[0] - n, max(0, (target_s - el) / max(el, 1e-3) * n)))
    n2 = (n2 // cores) * cores
    if n2 > 0:
        t0 = time.perf_counter()
        oracle.nn(ds.test[n:n + n2], ds.train, w, V=V, mode="pruned", envelopes_UL=(U, Lo))
        el += time.perf_counter() - t0
    total = n + n2
    # one thread on a small query subset (the single-core rate), ~target_s/3
    n1 = max(1, min(ds.test.shape[0], int(total / max(el, 1e-3) / cores * target_s / 3)))
    t0 = time.perf_counter()
    oracle.nn(ds.test[:n1], ds.train, w, V=V, mode="pruned", envelopes_UL=(U, Lo), threads=1)
    el1 = time.perf_counter() - t0
    return {"value": total / el, "unit": "queries/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"first {total} queries of the {ds.test.shape[0]} against all "
                      f"{ds.train.shape[0]} train series (fp64 oracle, paper-pruned mode ii, "
                      f"{el:.1f} s; envelopes precomputed, not timed, as P:583)",
            "one_thread": {"value": n1 / el1, "unit": "queries/s", "cores": 1,
                           "sample": f"first {n1} queries ({100.0 * n1 / ds.test.shape[0]:.2g} "
                                     f"% of the {ds.test.shape[0]}), {el1:.1f} s"}}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"



def run_reference(args, cfg, ds, w, V):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores = oracle.default_threads()
    U, Lo = oracle.envelopes(ds.train, w)
    nper = max(cores, int(args.ref_queries))
    Q = ds.test
    off = 0

    def step():
        nonlocal off
        sel = np.arange(off, off + nper) % Q.shape[0]
        off += nper
        oracle.nn(Q[sel], ds.train, w, V=V, mode="pruned", envelopes_UL=(U, Lo))

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = nper * args.steps / el
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(cfg, w, V, args.gpus),
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores,
                             "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{nper} queries per step (rolling through the "
                                       f"{Q.shape[0]}) against all {ds.train.shape[0]} "
                                       "train series, fp64 oracle paper-pruned search"},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_json(cfg, w, V, gpus):
    n, q, L = cfg.n_train, cfg.n_test, cfg.L
    lb_bytes = q * ((n + 3) // 4 * 4) * 4
    ser_bytes = n * L * 4 * 3
    big = lb_bytes + ser_bytes > 126 * 2 ** 20
    return {"workload": f"config{cfg.idx}_{cfg.name}", "n_train": n, "n_test": q, "L": L,
            "w": w, "V": V, "classes": cfg.classes,
            "l2": (f"inputs larger than L2 ({lb_bytes / 1e9:.2f} GB bound matrix + "
                   f"{ser_bytes / 1e6:.0f} MB series/envelopes per step)" if big else
                   f"working set {(lb_bytes + ser_bytes) / 1e6:.0f} MB fits the 126 MB L2 "
                   "(small config; not flushed)"),
            "parallelism": f"train-sharded x{gpus}, queries replicated, int64 MIN allreduce"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--queries", type=int, default=None, help="override Q (debug only)")
    ap.add_argument("--train", type=int, default=None, help="override N (debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-queries", type=int, default=0)
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded path (NCCL process group, seed exchange, 3-step MIN "
                         "combine) even at N=1 -- exercises the N>1 code on one GPU")
    args = ap.parse_args()

    cfg = datagen.CONFIGS[args.config]
    w = cfg.windows()[0] if args.config != 1 else datagen.window_from_percent(10, cfg.L)
    V = cfg.Vs[-1] if args.config not in (1,) else 5
    ds = datagen.make_dataset(args.config, n_train=args.train, n_test=args.queries)
    if args.impl == "reference":
        run_reference(args, cfg, ds, w, V)
        return

    import torch
    import torch.distributed as dist

    from paper_1808_09617_b200 import build as nbuild
    from paper_1808_09617_b200 import nndtw
    from paper_1808_09617_b200.dist import classify_sharded, shard_range

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or args.sharded
    if sharded:
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29513")
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    if rank == 0:
        nbuild.build()
    if world > 1:
        dist.barrier()
    lib = nndtw.load()
    if lib.nndtw_check_device() != 0:
        raise SystemExit("libnndtw requires an sm_100 (B200) device")
    N, L = ds.train.shape
    Q = ds.test.shape[0]
    lo, hi = shard_range(N, rank, world)
    train_h = torch.from_numpy(np.ascontiguousarray(ds.train[lo:hi])).pin_memory()
    test_h = torch.from_numpy(ds.test).pin_memory()
    labels_h = torch.from_numpy(ds.train_labels).pin_memory()
    train_d = train_h.to(dev)
    test_d = test_h.to(dev)
    labels_d = labels_h.to(dev)
    stream = torch.cuda.current_stream(dev)

    acc = {"ms_lb": 0.0, "ms_dtw": 0.0, "ms_lb_bridge": 0.0, "bridge_pairs": 0,
           "cells": 0, "lb_pairs": 0, "dtw_calls": 0,
           "survivors": 0, "near_tie_pairs": 0, "dtw_abandoned": 0}

    env_ev = []
    acc_env = [0.0]

    def step(stats):
        if stats:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(stream)
        model = nndtw.Model(train_d, labels_d[lo:hi], w, V, index_base=lo, check=False)
        if stats:
            ev[1].record(stream)
            env_ev.append(ev)
        if not sharded:
            pred = nndtw.classify(model, test_d, stats=stats, check=False)
        else:
            pred = classify_sharded(model, test_d, labels_d, stats=stats)
        if stats and pred.stats:
            for k in acc:
                acc[k] += pred.stats[k]
        return pred

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize(dev)

    # ---- timed region (device-side timing, max over ranks) -----------------------------
    sampler = ClockSampler(local) if rank == 0 else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    if sampler:
        sampler.start()
        time.sleep(0.3)
    l0 = nndtw.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        pred = step(True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = nndtw.launch_count() - l0
    acc_env_ms = sum(a.elapsed_time(b) for a, b in env_ev)
    env_bytes = (hi - lo) * L * 12.0  # read x, write U and L (S1 algorithmic bytes)
    # S1 launch duration: the in-step events above also hold the host-side gap before the
    # launch (the GPU idles while Python builds the Model), which is a large share of a
    # 0.15 ms kernel; so the kernel is also timed here as 20 back-to-back launches of the same
    # call on the same stream (inputs > L2, so no cache reuse between launches)
    env_reps = 20
    eU = torch.empty_like(train_d)
    eL = torch.empty_like(train_d)
    ek = torch.empty((hi - lo, 4), dtype=torch.int32, device=dev)
    est = nndtw._stream(stream)

    def env_launch():
        rc = lib.nndtw_envelopes(nndtw._ptr(train_d), hi - lo, L, w, nndtw._ptr(eU),
                                 nndtw._ptr(eL), nndtw._ptr(ek), est)
        assert rc == 0, rc
    env_launch()
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(env_reps):
        env_launch()
    g1.record(stream)
    torch.cuda.synchronize(dev)
    env_launch_ms = g0.elapsed_time(g1) / env_reps
    del eU, eL, ek
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms, float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms, launches = float(tmax[0]), int(tsum[1])
        a = torch.tensor([acc["ms_dtw"], acc["ms_lb"], float(acc["cells"]),
                          float(acc["lb_pairs"]), float(acc["dtw_calls"]), acc["ms_lb_bridge"],
                          float(acc["bridge_pairs"])],
                         dtype=torch.float64, device=dev)
        dist.all_reduce(a, op=dist.ReduceOp.SUM)
        acc_tot = {"ms_dtw": float(a[0]), "ms_lb": float(a[1]), "cells": float(a[2]),
                   "lb_pairs": float(a[3]), "dtw_calls": float(a[4]),
                   "ms_lb_bridge": float(a[5]), "bridge_pairs": float(a[6])}
    else:
        acc_tot = dict(acc)
    acc_tot["ms_dtw"] = acc_tot["ms_dtw"] / world
    acc_tot["ms_lb"] = acc_tot["ms_lb"] / world
    acc_tot["ms_lb_bridge"] = acc_tot["ms_lb_bridge"] / world
    value = Q * args.steps / (ms / 1e3)

    # ---- per-level prune counters (one untimed call; the level pass is not in the step) ----
    levels = None
    adapt_env = os.environ.get("NNDTW_ADAPT")
    if not sharded:
        model_l = nndtw.Model(train_d, labels_d[lo:hi], w, V, index_base=lo, check=False)
        st_l = nndtw.classify(model_l, test_d, stats=True, check=False, level_stats=True).stats
        levels = {k: st_l[k] for k in ("pruned_kim", "pruned_bands", "pruned_keogh",
                                       "survivors", "dtw_fallback")}
        # the survivor round's cells without the band-limited S4 pass (DESIGN.md "S4 band-limited
        # pass"): the full-window work the same answer takes, for the full-window-equivalent rate
        os.environ["NNDTW_ADAPT"] = "0"
        try:
            st_f = nndtw.classify(model_l, test_d, stats=True, check=False).stats
        finally:
            if adapt_env is None:
                del os.environ["NNDTW_ADAPT"]
            else:
                os.environ["NNDTW_ADAPT"] = adapt_env
        levels["cells_full_window"] = st_f["cells"]
        del model_l

    # ---- e2e through the public API with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e:
        def e2e_step():
            tr = train_h.to(dev, non_blocking=True)
            te = test_h.to(dev, non_blocking=True)
            lb_ = labels_h.to(dev, non_blocking=True)
            model = nndtw.Model(tr, lb_[lo:hi], w, V, index_base=lo)
            if not sharded:
                pred = nndtw.classify(model, te)
            else:
                pred = classify_sharded(model, te, lb_)
            return pred.idx.cpu(), pred.label.cpu(), pred.dist.cpu()
        e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        ke = max(1, min(args.steps, 3))
        for _ in range(ke):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = f0.elapsed_time(f1)
        if world > 1:
            te_ = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(te_, op=dist.ReduceOp.MAX)
            ems = float(te_[0])
        h2d = train_h.numel() * 4 + test_h.numel() * 4 + labels_h.numel() * 4
        d2h = Q * (8 + 4 + 4)
        e2e = {"value": Q * ke / (ems / 1e3), "unit": "queries/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    if rank != 0:
        if sharded:
            dist.barrier()
            dist.destroy_process_group()
        return

    pk, src = peaks()
    num_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    peak_cells = dtw_cell_peak_gcups(num_sms, sm_mhz)
    dtw_gcups = acc_tot["cells"] / (acc_tot["ms_dtw"] * 1e-3) / 1e9 / world \
        if acc_tot["ms_dtw"] > 0 else 0.0
    # per-GPU dominant-kernel figure: each rank's cells / its own DTW kernel time
    lb_cols = (L - 2 * min(L // 2, V))
    lb_rate = (acc_tot["lb_pairs"] * lb_cols / (acc_tot["ms_lb"] * 1e-3) / 1e9 / world
               if acc_tot["ms_lb"] > 0 else 0.0)
    lb_peak = lb_pair_col_peak(num_sms, sm_mhz)
    dominant = "dtw" if acc_tot["ms_dtw"] >= acc_tot["ms_lb"] else "lb"
    traffic = ncu_traffic()
    dtw_kernel = lib.nndtw_dtw_kernel_name(L, w).decode()  # the kernel dispatch_dtw runs
    wb = int(lib.nndtw_band_limited_window(L, w))
    dtw_label = (f"k_dtw_band band-limited pass (wb={wb}) + {dtw_kernel} full-window pass for "
                 f"the survivors it sends back (S4 survivor round)" if wb >= 0 else
                 f"{dtw_kernel} (S4 survivor round)")
    roof_dtw = {"kernel": dtw_label, "bound": "alu",
                "achieved": dtw_gcups, "peak": peak_cells, "unit": "Gcells/s",
                "frac": dtw_gcups / peak_cells if peak_cells else None,
                "traffic": traffic.get(dtw_kernel, {}).get("bytes_per_launch")
                if args.config == 2 else None,
                "peak_source": f"{num_sms} SMs x 64 cells/clk (FMNMX3 at 16 lanes/clk/SMSP, "
                               f"tools/pipebench.cu) x {sm_mhz:.0f} MHz ({src})",
                "ms_per_step": acc_tot["ms_dtw"] / args.steps}
    if levels and levels.get("cells_full_window") and acc_tot["ms_dtw"] > 0 and \
            levels["cells_full_window"] > 1.01 * acc_tot["cells"] / args.steps:
        # band-limited pass on: the cells it computes are fewer than the full window's; the
        # same answer over the full window takes cells_full_window (untimed run, pass off)
        eq = levels["cells_full_window"] / (acc_tot["ms_dtw"] / args.steps * 1e-3) / 1e9 / world
        roof_dtw["full_window_equivalent"] = {
            "cells_per_step": levels["cells_full_window"], "achieved": eq,
            "frac": eq / peak_cells if peak_cells else None,
            "note": "full-window survivor-round cells (NNDTW_ADAPT=0, untimed) / the timed "
                    "survivor round; achieved/frac above count the cells actually computed"}
    lb_bytes = (Q * L + (hi - lo) * (2 * L + 2 * min(L // 2, V)) + Q * (hi - lo)) * 4.0
    two_stage = acc_tot["ms_lb_bridge"] > 0 and acc_tot["bridge_pairs"] < acc_tot["lb_pairs"]
    if two_stage:
        # two-stage S2: stage A (Kim + bands, every pair) and the bridge for the pairs the
        # partial cascade kept; the roofline figure is the bridge kernel's own pair-columns/s
        br_rate = (acc_tot["bridge_pairs"] * lb_cols / (acc_tot["ms_lb_bridge"] * 1e-3) / 1e9
                   / world)
        roof_lb = {"kernel": "k_lb_sparse (S2 stage B: LB_Keogh bridge on the pairs LB_Kim + "
                             "Algorithm 1's bands kept)", "bound": "alu",
                   "achieved": br_rate, "peak": lb_peak, "unit": "G pair-columns/s",
                   "frac": br_rate / lb_peak if lb_peak else None,
                   "traffic": traffic.get("k_lb_sparse", {}).get("bytes_per_launch")
                   if args.config == 2 else None,
                   "bridge_pairs_per_step": acc_tot["bridge_pairs"] / args.steps,
                   "bridge_fraction": acc_tot["bridge_pairs"] / max(acc_tot["lb_pairs"], 1),
                   "peak_source": f"{num_sms} SMs x 42.7 pair-cols/clk (3 FMA-pipe ops each) x "
                                  f"{sm_mhz:.0f} MHz ({src})",
                   "ms_per_step": acc_tot["ms_lb_bridge"] / args.steps,
                   "ms_s2_per_step": acc_tot["ms_lb"] / args.steps}
        # the bridge streams every listed pair's query row (L floats) out of L2: its second
        # roof is the L2 -> SM read rate for 2 KB rows (tools/l2_roof.cu on B200: 18.3 TB/s at
        # 16 warps/SM, 20.3 TB/s at 32; profiles/round2d_l2_roof.txt)
        if acc_tot["ms_lb_bridge"] > 0:
            l2_gbs = (acc_tot["bridge_pairs"] * L * 4 / (acc_tot["ms_lb_bridge"] * 1e-3) / 1e9
                      / world)
            roof_lb["l2_rows"] = {"achieved": l2_gbs, "peak": L2_ROW_GBS, "unit": "GB/s",
                                  "frac": l2_gbs / L2_ROW_GBS,
                                  "peak_source": "tools/l2_roof.cu, 2 KB rows, 16 warps/SM "
                                                 "(measured, B200)"}
    else:
        roof_lb = None
    roof_lb = roof_lb or {"kernel": "k_lb_tile (S2 cascade)", "bound": "alu", "achieved": lb_rate,
               "peak": lb_peak, "unit": "G pair-columns/s",
               "frac": lb_rate / lb_peak if lb_peak else None,
               "traffic": traffic.get("k_lb_tile", {}).get("bytes_per_launch")
               if args.config == 2 else None,
               "hbm_gbs": (lb_bytes / (acc_tot["ms_lb"] / args.steps * 1e-3) / 1e9
                           if acc_tot["ms_lb"] > 0 else None),
               "peak_source": f"{num_sms} SMs x 42.7 pair-cols/clk (3 FMA-pipe ops each) x "
                              f"{sm_mhz:.0f} MHz ({src})",
               "ms_per_step": acc_tot["ms_lb"] / args.steps}
    hbm = float(pk.get("hbm_gbs", 6650.0))
    env_gbs = env_bytes / (env_launch_ms * 1e-3) / 1e9 if env_launch_ms > 0 else None
    env_kernel = envelope_kernel(L, w)
    roof_env = {"kernel": f"{env_kernel} (S1)", "bound": "hbm", "achieved": env_gbs, "peak": hbm,
                "unit": "GB/s", "frac": env_gbs / hbm if env_gbs else None,
                "traffic": traffic.get(env_kernel, {}).get("bytes_per_launch")
                if args.config == 2 else None,
                "algorithmic_bytes": env_bytes,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "ms_per_launch": env_launch_ms,
                "timing": f"{env_reps} back-to-back launches after the timed region (CUDA "
                          "events); ms_per_step is the in-step event time, host gap included",
                "ms_per_step": acc_env_ms / args.steps}
    line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (datagen.py, BASELINE.json configs[%d])" %
            args.config, "config": config_json(cfg, w, V, world),
            "roofline": roof_dtw if dominant == "dtw" else roof_lb,
            "roofline_other": roof_lb if dominant == "dtw" else roof_dtw,
            "roofline_envelopes": roof_env,
            "dtw_gcups": dtw_gcups,
            "effective_gcups": Q * N * (L * (2 * w + 1) - w * (w + 1)) /
            (ms / args.steps * 1e-3) / 1e9,
            "counters_per_step": {**{k: acc_tot[k] / args.steps for k in
                                     ("lb_pairs", "dtw_calls", "cells")}, **(levels or {})},
            "gpu_launches": launches, "clocks": clocks, "e2e": e2e}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_oracle(ds, w, V)
    print(json.dumps(line), flush=True)
    if sharded:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
