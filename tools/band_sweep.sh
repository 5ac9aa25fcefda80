#!/bin/bash
# Sweep the band kernel's slot width R and packing per (L, w): raw GCUPS via tools/dtw_rate.py.
#   bash tools/band_sweep.sh "L:w:P ..." "R list" > gpurun_out/band_sweep.txt
shapes=${1:-"512:103:200000"}
rs=${2:-"8 10 12 14 16 18 20 22 24 26 28 30 32"}
for s in $shapes; do
  for r in $rs; do
    for pk in 0 1; do
      out=$(NNDTW_VERBOSE=1 NNDTW_BAND_R=$r NNDTW_PACK=$pk python tools/dtw_rate.py $s 2>&1)
      cfg=$(echo "$out" | grep "nndtw band" | tail -1 | sed 's/.*-> //')
      g=$(echo "$out" | grep GCUPS | sed 's/.*ms  //')
      [ -n "$cfg" ] && echo "$s R=$r pack=$pk | $cfg | $g"
    done
  done
done
