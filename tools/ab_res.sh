#!/bin/bash
# A/B timing of the cfg1 resident kernel for alternative builds (dev tool): bash tools/ab_res.sh lib1.so lib2.so ...
# (per-L table on, 3 alternating rounds so clock drift shows)
for r in 1 2 3; do
  for L in "$@"; do
    FIF_LIB_PATH=$L python tools/time_variant.py $L 4096 4096 --eig 2>&1 | tail -1
  done
done
