set -u
O=gpurun_out/r2o; mkdir -p $O
for r in 1 2; do for L in variants/prev.so paper_1802_01359_b200/libfif_b200.so; do
  FIF_LIB_PATH=$L python tools/time_variant.py $L 262144 1024 --eig --f32 2>&1 | tail -1
done; done 2>&1 | tee $O/ab.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_options.py tests/test_gpu_fuzz.py -m gpu -q -rfE > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
