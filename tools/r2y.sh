set -u
O=gpurun_out/r2y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_streamed.py -m gpu -x -q -rfE > $O/tests1.log 2>&1; echo "streamed tests rc=$?"; tail -3 $O/tests1.log
for r in 1 2; do
  timeout 300 python tools/run_plan.py --config cfg3 --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|cfg3 |"
  timeout 300 python tools/run_plan.py --config cfg2 --regime 2 --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|cfg2-streamed |"
  for n in 131072 49152 1048576; do
  timeout 300 python tools/run_plan.py --config cfg4 --n $n --batch $((268435456 / n)) --reps 3 2>&1 | tail -1 | cut -c1-40 | sed "s|^|n=$n |"
  done
done 2>&1 | tee $O/ab.txt
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -m gpu -q -rfE -x > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
python bench.py --config cfg3 --steps 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for n in 131072 1048576 49152 81920; do
  python bench.py --config cfg4 --n $n --steps 5 --no-cpu --no-e2e > $O/bench_cfg4_$n.json 2> $O/bench_cfg4_$n.err
done
echo done
