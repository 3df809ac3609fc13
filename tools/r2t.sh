set -u
O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_streamed.py -m gpu -x -q -rfE -k "bulk_copy" > $O/tests1.log 2>&1; echo "bulk tests rc=$?"; tail -3 $O/tests1.log
for r in 1 2; do for RM in 0 1 2; do
  FIF_ST_RM=$RM timeout 300 python tools/run_plan.py --config cfg3 --reps 3 2>&1 | tail -1 | sed "s|^|RM=$RM cfg3 |"
  for n in 131072 49152 1048576; do
  FIF_ST_RM=$RM timeout 300 python tools/run_plan.py --config cfg4 --n $n --batch $((268435456 / n)) --reps 3 2>&1 | tail -1 | sed "s|^|RM=$RM n=$n |"
  done
done; done 2>&1 | tee $O/ab.txt
