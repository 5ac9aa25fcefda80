"""bench.py's host-side pieces on CPU: the roofline peaks follow DESIGN.md §7's pipe model, the
config block names the workload, and the reference arm's JSON line has the contract's keys
(run on a tiny sample, CPU oracle only)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_peaks_follow_pipe_model():
    import bench
    # 148 SMs x 64 cells/clk x 1965 MHz; 148 x 128/3 pair-columns/clk x 1965 MHz
    assert bench.dtw_cell_peak_gcups(148, 1965.0) == pytest.approx(148 * 64 * 1.965)
    assert bench.lb_pair_col_peak(148, 1965.0) == pytest.approx(148 * 128 / 3 * 1.965)


def test_config_json_names_workload():
    import bench
    import datagen
    cfg = datagen.CONFIGS[2]
    c = bench.config_json(cfg, 103, 5, 8)
    assert c["workload"] == "config2_large_search" and c["w"] == 103 and c["V"] == 5
    assert "larger than L2" in c["l2"] and "x8" in c["parallelism"]
    c0 = bench.config_json(datagen.CONFIGS[0], 13, 5, 1)
    assert "fits the 126 MB L2" in c0["l2"]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "0", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
