"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [--json out.json]

`launches`: per-kernel launch counts, total device time and share of the launch list
(`--metrics gpu__time_duration.sum`, cold-cache and serialised: compare SHARES).
`full`: per captured kernel the counters the roofline uses (duration, DRAM bytes, issue
utilisation, pipe utilisation, warps, registers, stall breakdown).
"""
import collections
import csv
import io
import json
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
             "ms": 1.0, "second": 1e3, "s": 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {v / T * 100:.1f}% |")
    with open(out, "w") as f:
        f.write(f"# Launch list ({path})\n\n`ncu --metrics gpu__time_duration.sum "
                "--clock-control none` over the default `python bench.py` command "
                "(cold-cache, serialised: compare shares, not absolutes).\n\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed.avg.per_cycle_elapsed", "IPC per SM (max 4)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def full(path, out, jpath=None):
    raw = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = dict(zip(h, rows[1]))
    res = []
    md = [f"# Full ncu capture ({path})\n"]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"]
        rec = {"kernel": name}
        md.append(f"## `{name}`\n")
        md.append("| counter | value |\n|---|---|")
        for k, label in KEYS:
            v = d.get(k, "")
            u = units.get(k, "")
            rec[k] = v
            md.append(f"| {label} (`{k}`) | {v} {u} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0)
                  for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = sorted(stalls.items(), key=lambda x: -x[1])[:8]
        md.append("\nwarp-state samples: " + ", ".join(f"{k} {v / tot * 100:.1f}%"
                                                      for k, v in top) + "\n")
        rec["stalls"] = {k: v / tot for k, v in top}
        res.append(rec)
    with open(out, "w") as f:
        f.write("\n".join(md) + "\n")
    if jpath:
        json.dump(res, open(jpath, "w"), indent=1)
    print("\n".join(md))


def traffic(path, out):
    """profiles/ncu_traffic.json: dram read+write bytes of the longest captured launch of each
    kernel (bench.py reads it for roofline.traffic)."""
    raw = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    units = dict(zip(h, rows[1]))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    tmult = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6,
             "us": 1e-3, "ms": 1.0, "s": 1e3}
    best = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        name = name.split("::")[-1]
        ms = float(d["gpu__time_duration.sum"]) * tmult[units["gpu__time_duration.sum"]]
        b = sum(float(d[k]) * mult[units[k]] for k in ("dram__bytes_read.sum",
                                                        "dram__bytes_write.sum"))
        if b != b:  # metrics not collected for this launch
            continue
        if name not in best or ms > best[name]["ms"]:
            best[name] = {"ms": ms, "bytes_per_launch": b, "report": path}
    json.dump(best, open(out, "w"), indent=1)
    print(json.dumps(best, indent=1))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    elif mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        jp = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
        full(sys.argv[2], sys.argv[3], jp)
