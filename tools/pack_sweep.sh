#!/bin/bash
# Packed vs unpacked band kernel at the chooser's layout, per (L, w): raw GCUPS.
SHAPES=${1:-"128:13:800000 256:26:400000 256:52:300000 256:128:150000 256:255:100000 300:3:600000 300:15:600000 300:30:300000 300:60:200000 300:90:150000 300:120:120000 300:150:100000 300:180:100000 300:210:80000 300:240:80000 300:270:70000 300:299:60000 512:103:200000"}
for s in $SHAPES; do
  for pk in 0 1; do
    out=$(NNDTW_VERBOSE=1 NNDTW_PACK=$pk python tools/dtw_rate.py $s 2>&1)
    cfg=$(echo "$out" | grep "nndtw band" | tail -1 | sed 's/.*-> //')
    g=$(echo "$out" | grep GCUPS | sed 's/.*ms  //')
    echo "$s pack=$pk | $cfg | $g"
  done
done
