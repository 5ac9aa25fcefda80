"""Summarise an ncu report: key counters, stall mix, and per-opcode stall attribution.

  python tools/ncu_stalls.py gpurun_out/prof.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "sm__inst_executed.avg.per_cycle_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:70s} {v[i]} {rows[1][i]}")
items = [(h[i], v[i]) for i in range(len(h))
         if "pcsamp_warps_issue_stalled" in h[i] and not h[i].endswith("not_issued")]
tot = sum(float(x or 0) for _, x in items)
print("stall mix:", ", ".join(f"{n.split('stalled_')[1]} {float(x) / tot * 100:.1f}%"
                             for n, x in sorted(items, key=lambda t: -float(t[1] or 0))[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
idx = {c: i for i, c in enumerate(h)}
cols = ["stall_selected", "stall_not_selected", "stall_dispatch", "stall_wait", "stall_math",
        "stall_short_sb", "stall_long_sb", "stall_barrier", "stall_mio"]
agg = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    op = r[idx["Source"]].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    for c in cols:
        try:
            agg[o][c] += float(r[idx[c]] or 0)
        except (KeyError, ValueError):
            pass
    try:
        agg[o]["n"] += float(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        pass
tot = sum(sum(x[c] for c in cols) for x in agg.values()) or 1.0
for o, x in sorted(agg.items(), key=lambda kv: -sum(kv[1][c] for c in cols))[:12]:
    print(f"{o:8s} exec={x['n']:.3g} " + " ".join(f"{c[6:]}={x[c] / tot * 100:.1f}"
                                                 for c in cols if x[c] / tot > 0.002))
