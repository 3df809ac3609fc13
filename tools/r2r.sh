set -u
O=gpurun_out/r2r; mkdir -p $O
for r in 1 2; do for L in variants/prev.so paper_1802_01359_b200/libfif_b200.so; do
  FIF_LIB_PATH=$L timeout 300 python tools/run_plan.py --config cfg3 --reps 3 2>&1 | tail -1 | sed "s|^|$L cfg3 |"
  for n in 131072 49152; do
  FIF_LIB_PATH=$L timeout 300 python tools/run_plan.py --config cfg4 --n $n --batch $((268435456 / n)) --reps 3 2>&1 | tail -1 | sed "s|^|$L n=$n |"
  done
done; done 2>&1 | tee $O/ab.txt
timeout 1500 python -m pytest tests/test_gpu_streamed.py tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py tests/test_gpu_dist.py tests/test_gpu_workspace.py -m gpu -q -rfE > $O/tests.log 2>&1; echo "tests rc=$?"; tail -4 $O/tests.log
