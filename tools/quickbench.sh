#!/bin/bash
# quick GPU check: fast parity tests + a short config-2 bench summary line
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m "gpu and not slow" --timeout 300 -p no:cacheprovider 2>&1 | tail -1
python bench.py --steps 3 --warmup 2 --no-cpu-baseline "$@" > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
r, o = d["roofline"], d["roofline_other"]
print(f"q/s={d['value']:.0f} ms/step={d['ms_per_step']:.1f} dtw={r['ms_per_step']:.1f}ms "
      f"{r['achieved']:.0f}{r['unit']} frac={r['frac']:.3f} lb={o['ms_per_step']:.1f}ms "
      f"frac={o['frac']:.3f} e2e={d['e2e']['value']:.0f} calls={d['counters_per_step']}")
PY
