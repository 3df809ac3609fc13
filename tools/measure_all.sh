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
FIF_DIST_PEER=1 python bench.py --config cfg3 --emulate 8 --steps 3 --no-cpu --no-e2e > $O/bench_cfg3_emul8_peer.json 2> $O/bench_cfg3_emul8_peer.err
for n in 1024 16384 131072 1048576 49152 81920; do
  python bench.py --config cfg4 --n $n --steps 5 --no-cpu --no-e2e > $O/bench_cfg4_$n.json 2> $O/bench_cfg4_$n.err
done
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; tail -c 300 $O/bench_reference.json
echo measure_all done
