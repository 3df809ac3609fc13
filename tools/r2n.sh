#!/bin/bash
# Round-2 ncu session (run under gpurun from the repo root): launch lists + one full capture.
set -u
O=gpurun_out/r2n; mkdir -p $O
LM="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-secondary > $O/plain_b1.log 2>&1 && \
  ncu $LM -c 400 --log-file $O/launches_bench_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-secondary > $O/ncu_b1.log 2>&1; echo "b1 $?"
python tools/run_plan.py --config cfg2 --batch 512 --reps 2 > $O/plain_c2.log 2>&1 && \
  ncu $LM -s 1 -c 1 --log-file $O/launches_cfg2.csv python tools/run_plan.py --config cfg2 --batch 512 --reps 2 > $O/ncu_c2.log 2>&1; echo "c2 $?"
python tools/run_plan.py --config cfg3 --reps 2 > $O/plain_c3.log 2>&1 && \
  ncu $LM -s 76 -c 76 --log-file $O/launches_cfg3.csv python tools/run_plan.py --config cfg3 --reps 2 > $O/ncu_c3.log 2>&1; echo "c3 $?"
python tools/run_plan.py --config cfg4 --n 131072 --batch 2048 --reps 2 > $O/plain_c4.log 2>&1 && \
  ncu $LM -s 260 -c 260 --log-file $O/launches_cfg4_131072.csv python tools/run_plan.py --config cfg4 --n 131072 --batch 2048 --reps 2 > $O/ncu_c4.log 2>&1; echo "c4 $?"
python tools/run_plan.py --config cfg4 --n 1024 --batch 262144 --reps 2 --eig > $O/plain_f32.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fif_resident_kernel -s 1 -c 1 -o $O/full_f32_1024 \
    python tools/run_plan.py --config cfg4 --n 1024 --batch 262144 --reps 2 --eig > $O/ncu_f32.log 2>&1; echo "f32 $?"
ls $O
