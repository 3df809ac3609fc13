set -u
O=gpurun_out/r2i; mkdir -p $O
python tools/run_plan.py --config cfg4 --n 1024 --batch 262144 --reps 2 --eig > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fif_resident_kernel -s 1 -c 1 -o $O/full_f32_1024 \
  python tools/run_plan.py --config cfg4 --n 1024 --batch 262144 --reps 2 --eig > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/full_f32_1024.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
cat $O/plain.log
