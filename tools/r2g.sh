set -u
O=gpurun_out/r2g; mkdir -p $O
for r in 1 2; do for L in variants/old.so paper_1802_01359_b200/libfif_b200.so; do
  FIF_LIB_PATH=$L timeout 300 python tools/run_plan.py --config cfg2 --batch 512 --reps 4 2>&1 | tail -1 | sed "s|^|$L |"
done; done 2>&1 | tee $O/ab.txt
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_determinism.py -m gpu -x -q -rfE > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
