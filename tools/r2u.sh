set -u
# A/B of the tensor-map tiles on fp64 streamed geometries, then ncu --set full of the streamed kernels of
# config 3 (one IMF's kernels in the steady state; ONE ncu invocation per gpurun call)
O=gpurun_out/r2u; mkdir -p $O
for r in 1 2; do for RM in 0 2; do
  FIF_ST_RM=$RM timeout 300 python tools/run_plan.py --config cfg2 --regime 2 --reps 3 2>&1 | tail -1 | sed "s|^|RM=$RM cfg2-streamed |"
  FIF_ST_RM=$RM timeout 300 python tools/run_plan.py --config cfg3 --n 16777216 --reps 3 2>&1 | tail -1 | sed "s|^|RM=$RM cfg3-2^24 |"
  FIF_ST_RM=$RM timeout 300 python tools/run_plan.py --config cfg1 --n 1048576 --batch 64 --regime 2 --reps 3 2>&1 | tail -1 | sed "s|^|RM=$RM f64-2^20x64 |"
done; done 2>&1 | tee $O/ab.txt
FIF_ST_RM=2 python tools/run_plan.py --config cfg3 --reps 1 > $O/plain3.log 2>&1 && \
FIF_ST_RM=2 ncu --set full --clock-control none --import-source on -k regex:"k_col|k_rows_inv" -s 6 -c 4 -o $O/full_cfg3 \
  python tools/run_plan.py --config cfg3 --reps 1 > $O/ncu_f3.log 2>&1
echo "ncu rc=$?"; ls -la $O
