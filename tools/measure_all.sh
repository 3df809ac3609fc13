#!/bin/bash
# One GPU session of measurements for profiles/ (run under gpurun from the repo root).
set -u
O=gpurun_out/m
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err; tail -c 300 $O/bench_cfg1.json
python bench.py --config cfg2 --steps 5 --no-cpu > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --config cfg3 --steps 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config cfg3 --emulate 8 --steps 3 --no-cpu --no-e2e > $O/bench_cfg3_emul8.json 2> $O/bench_cfg3_emul8.err
for n in 1024 16384 131072 1048576 49152 81920; do
  python bench.py --config cfg4 --n $n --steps 5 --no-cpu --no-e2e > $O/bench_cfg4_$n.json 2> $O/bench_cfg4_$n.err
done
# launch lists (cold-cache, serialised: shares, not absolutes) of one step after the warm-up
python tools/run_plan.py --config cfg2 --reps 1 > $O/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 65 -c 65 --csv \
    --log-file $O/launches_cfg2.csv python tools/run_plan.py --config cfg2 --reps 2 > $O/ncu_l2.log 2>&1
python tools/run_plan.py --config cfg3 --reps 1 > $O/plain3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 76 -c 76 --csv \
    --log-file $O/launches_cfg3.csv python tools/run_plan.py --config cfg3 --reps 2 > $O/ncu_l3.log 2>&1
python tools/run_plan.py --config cfg1 --reps 1 > $O/plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 2 -c 2 --csv \
    --log-file $O/launches_cfg1.csv python tools/run_plan.py --config cfg1 --reps 3 > $O/ncu_l1.log 2>&1
# full captures: the resident kernel (cfg1) and the two heaviest streamed kernels (cfg2)
ncu --set full --clock-control none --import-source on -k regex:fif_resident_kernel -s 1 -c 1 -o $O/full_resident \
    python tools/run_plan.py --config cfg1 --reps 2 > $O/ncu_f1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_col|k_rows_inv" -s 3 -c 2 -o $O/full_cfg2 \
    python tools/run_plan.py --config cfg2 --reps 1 > $O/ncu_f2.log 2>&1
echo measure_all done
