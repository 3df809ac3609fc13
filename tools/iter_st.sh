#!/bin/bash
# One GPU iteration on the streamed regime (dev tool, run under gpurun from the repo root):
# streamed + fuzz tests, config 2 / 3 bench lines (no cpu/e2e), then the launch list of one cfg2 call.
set -u
O=gpurun_out/st
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_streamed.py tests/test_gpu_fuzz.py tests/test_gpu_workspace.py -m gpu -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
for c in cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err
  python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c ms',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
if [ "${NCU:-1}" = "1" ]; then
  python tools/run_plan.py --config cfg2 --reps 1 > $O/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -s 65 -c 65 --log-file $O/launches_cfg2.csv python tools/run_plan.py --config cfg2 --reps 2 > $O/ncu.log 2>&1
  echo "ncu rc=$?"
  python tools/launches.py $O/launches_cfg2.csv 2>/dev/null | head -12
fi
