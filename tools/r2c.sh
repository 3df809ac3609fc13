set -u
O=gpurun_out/r2c; mkdir -p $O
bash tools/ab_res.sh variants/old.so paper_1802_01359_b200/libfif_b200.so variants/noltab.so 2>&1 | tee $O/ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_options.py tests/test_gpu_fuzz.py -m gpu -x -q -rfE > $O/tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/tests.log
