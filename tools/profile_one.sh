#!/bin/bash
# ncu captures for profiles/, ONE ncu invocation per gpurun call (run from the repo root):
#   bash tools/profile_one.sh launches1|launches2|launches3|full1|full2
set -u
O=gpurun_out/m
mkdir -p $O
LM="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
case "$1" in
  launches1) python tools/run_plan.py --config cfg1 --reps 1 > $O/plain1.log 2>&1 && \
    ncu $LM -s 2 -c 2 --log-file $O/launches_cfg1.csv python tools/run_plan.py --config cfg1 --reps 3 > $O/ncu_l1.log 2>&1 ;;
  launches2) python tools/run_plan.py --config cfg2 --reps 1 > $O/plain2.log 2>&1 && \
    ncu $LM -s 65 -c 65 --log-file $O/launches_cfg2.csv python tools/run_plan.py --config cfg2 --reps 2 > $O/ncu_l2.log 2>&1 ;;
  launches3) python tools/run_plan.py --config cfg3 --reps 1 > $O/plain3.log 2>&1 && \
    ncu $LM -s 76 -c 76 --log-file $O/launches_cfg3.csv python tools/run_plan.py --config cfg3 --reps 2 > $O/ncu_l3.log 2>&1 ;;
  full1) python tools/run_plan.py --config cfg1 --reps 1 > $O/plain1.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:fif_resident_kernel -s 1 -c 1 -o $O/full_resident \
      python tools/run_plan.py --config cfg1 --reps 2 --eig > $O/ncu_f1.log 2>&1 ;;
  full2) python tools/run_plan.py --config cfg2 --reps 1 > $O/plain2.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"k_col|k_rows_inv" -s 3 -c 2 -o $O/full_cfg2 \
      python tools/run_plan.py --config cfg2 --reps 1 > $O/ncu_f2.log 2>&1 ;;
esac
echo "profile_one $1 rc=$?"
