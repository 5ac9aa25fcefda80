#!/bin/bash
# Round-2 evidence set (one GPU): profile_round.sh's bench lines, launch list and full ncu capture
# of config 2, plus the config-1 grid / config-3 LOOCV table (tools/bench_configs.py) and the
# NN-DTW time-per-bound tables (tools/bound_table.py).
#   gpurun -- 'bash tools/profile_round2.sh round2b'
set -x
tag=${1:-round2}
mkdir -p gpurun_out
python -c "from paper_1808_09617_b200 import build; build.build()"
python tools/bench_configs.py --configs 1,3 > gpurun_out/${tag}_configs.jsonl 2> gpurun_out/${tag}_configs.err
python tools/bound_table.py --config 1 > gpurun_out/${tag}_bound_table_cfg1.md 2>&1
python tools/bound_table.py --config 2 --queries 1000 > gpurun_out/${tag}_bound_table_cfg2.md 2>&1
bash tools/profile_round.sh ${tag}
