#!/bin/bash
# The evidence behind profiles/<tag>_*: bench lines (config 2 with the oracle beside it, configs
# 0/1/4 without), the ncu launch list of the bench command and one full ncu capture of its top
# kernels.  Run on the GPU box (one GPU), e.g.
#   gpurun -- 'bash tools/profile_round.sh round1k'
# then summarise here:
#   python tools/ncu_summary.py launches gpurun_out/launches_<tag>.csv profiles/<tag>_launches.md
#   python tools/ncu_summary.py full gpurun_out/prof_<tag>.ncu-rep profiles/<tag>_full.md --json profiles/<tag>_full.json
#   python tools/ncu_summary.py traffic gpurun_out/prof_<tag>.ncu-rep profiles/ncu_traffic.json
set -x
tag=${1:-round}
mkdir -p gpurun_out
python bench.py > gpurun_out/${tag}_bench.log 2>&1
tail -1 gpurun_out/${tag}_bench.log > gpurun_out/${tag}_bench.json
for c in 0 1 4; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/${tag}_cfg$c.log 2>&1
  tail -1 gpurun_out/${tag}_cfg$c.log > gpurun_out/${tag}_bench_cfg$c.json
done
# launch list only after the same command exited 0 without ncu (above)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"k_dtw_band|k_lb_tile|k_lb_sparse|k_col_compact|k_list_compact|k_env_direct|k_compact|k_pad_rows" -c 12 -o gpurun_out/prof_${tag} \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
