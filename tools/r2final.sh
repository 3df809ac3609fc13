#!/bin/bash
# Final round-2 measurement pass (run under gpurun from the repo root): GPU tests, every bench line,
# then the ncu launch list of the default bench command.
set -u
bash tools/measure_all.sh
O=gpurun_out/m
LM="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $LM -c 400 --log-file $O/launches_bench_cfg1.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary > $O/ncu_bench.log 2>&1
echo "ncu launches rc=$?"
python tools/run_plan.py --config cfg3 --reps 1 > $O/plain3.log 2>&1 && \
timeout 600 ncu $LM -s 76 -c 76 --log-file $O/launches_cfg3.csv python tools/run_plan.py --config cfg3 --reps 2 > $O/ncu_l3.log 2>&1
echo "ncu cfg3 launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_col|k_rows_inv" -s 6 -c 4 -o $O/full_cfg3 \
  python tools/run_plan.py --config cfg3 --reps 1 > $O/ncu_f3.log 2>&1
echo "ncu cfg3 full rc=$?"
