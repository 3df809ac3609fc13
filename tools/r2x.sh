set -u
O=gpurun_out/r2x; mkdir -p $O
for r in 1 2; do
  timeout 300 python tools/run_plan.py --config cfg3 --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|cfg3 |"
  timeout 300 python tools/run_plan.py --config cfg2 --regime 2 --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|cfg2-streamed |"
  timeout 300 python tools/run_plan.py --config cfg3 --n 16777216 --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|cfg3-2^24 |"
  for n in 131072 49152 1048576; do
  timeout 300 python tools/run_plan.py --config cfg4 --n $n --batch $((268435456 / n)) --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|n=$n |"
  done
done 2>&1 | tee $O/ab.txt
