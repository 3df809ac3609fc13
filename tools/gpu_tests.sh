#!/bin/bash
# GPU test suite file by file, each under its own time limit (dev tool; run under gpurun from the repo root):
#   bash tools/gpu_tests.sh [file ...]     (default: every tests/test_gpu_*.py)
set -u
O=gpurun_out/gt
mkdir -p $O
FILES=${@:-$(ls tests/test_gpu_*.py)}
for f in $FILES; do
  b=$(basename $f .py)
  timeout ${T:-900} python -m pytest $f -m gpu -q -rfE -p no:cacheprovider > $O/$b.log 2>&1
  rc=$?
  echo "== $b rc=$rc $(tail -1 $O/$b.log)"
  grep -E "^(FAILED|ERROR)|parity floor" $O/$b.log | head -8
done
