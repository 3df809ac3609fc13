#!/bin/bash
# One GPU iteration on the resident kernel (dev tool, run under gpurun from the repo root):
# resident parity + options tests, the cfg1 bench line (no cpu/e2e), then one ncu --set full capture.
set -u
O=gpurun_out/it
mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_options.py -m gpu -x -q > $O/tests.log 2>&1; tail -3 $O/tests.log
python bench.py --no-cpu --no-e2e --steps 20 > $O/bench.json 2> $O/bench.err
python -c "import json;d=json.load(open('$O/bench.json'));print('ms',d['ms_per_step'],'frac',d['roofline']['frac'],'clk',d['clocks'])"
if [ "${NCU:-1}" = "1" ]; then
  python tools/run_plan.py --config cfg1 --reps 2 --eig > $O/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fif_resident_kernel -s 1 -c 1 -o $O/full \
    python tools/run_plan.py --config cfg1 --reps 2 --eig > $O/ncu.log 2>&1
  echo "ncu rc=$?"
fi
