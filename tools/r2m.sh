#!/bin/bash
# Round-2 measurement session (run under gpurun from the repo root): GPU tests, every bench line.
set -u
O=gpurun_out/r2m
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/gpu_tests.log
python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "bench rc=$?"
python bench.py --config cfg3 --steps 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
python bench.py --config cfg3 --emulate 8 --steps 3 --no-cpu --no-e2e > $O/bench_cfg3_emul8.json 2> $O/bench_cfg3_emul8.err
FIF_DIST_PEER=1 python bench.py --config cfg3 --emulate 8 --steps 3 --no-cpu --no-e2e > $O/bench_cfg3_emul8_peer.json 2> $O/bench_cfg3_emul8_peer.err
for n in 1024 16384 131072 1048576 49152 81920; do
  python bench.py --config cfg4 --n $n --steps 5 --no-cpu --no-e2e > $O/bench_cfg4_n$n.json 2> $O/bench_cfg4_n$n.err
done
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for f in $O/bench_*.json; do echo "$f $(python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d.get('ms_per_step'),d.get('value'),(d.get('roofline') or {}).get('frac'))" 2>&1)"; done
echo measure done
