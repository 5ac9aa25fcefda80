#!/bin/bash
# Share of the band kernel's warp time spent waiting for item setups (row copies), config 2:
# builds tools/_libnndtw_prof.so with -DNNDTW_PROFILE_SETUP (clock64 around the setup wait) and
# runs bench.py against it; the library prints setup_cycles / warp_cycles per classify call.
#   gpurun -- 'bash tools/setup_share.sh'
set -e
out=${TMPDIR:-/tmp}/nndtw_prof
mkdir -p $out
for f in abi envelopes lb dtw_band dtw_strip search bounds_next bounds_improved; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
    -cudart static -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr \
    -I include -DNNDTW_PROFILE_SETUP -c paper_1808_09617_b200/csrc/$f.cu -o $out/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a $out/*.o \
  -o tools/_libnndtw_prof.so -cudart static -Xlinker --no-undefined
NNDTW_LIB=tools/_libnndtw_prof.so timeout 300 python bench.py --steps 2 --warmup 1 \
  --no-cpu-baseline --no-e2e 2>&1 | grep -a "PROFILE_SETUP"
