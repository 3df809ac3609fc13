#!/bin/bash
# One GPU iteration on the cluster regime (dev tool): tests, config-2 timing (cluster vs streamed), launch list
set -u
O=gpurun_out/cl
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cluster.py -m gpu -q -x > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 300 python bench.py --config cfg2 --no-cpu --no-e2e --steps 5 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python -c "import json;d=json.load(open('$O/bench_cfg2.json'));print('cfg2 ms',round(d['ms_per_step'],3),'frac',round(d['roofline']['frac'],3),d['config']['regime'],d['config']['launch'])" 2>&1 | tail -1
tail -3 $O/bench_cfg2.err
