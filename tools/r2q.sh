set -u
O=gpurun_out/r2q; mkdir -p $O
python tools/run_plan.py --config cfg3 --reps 2 > $O/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_col" -s 30 -c 3 -o $O/full_col \
  python tools/run_plan.py --config cfg3 --reps 2 > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/full_col.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/full_col.ncu-rep --page source --csv --print-source sass > $O/src.csv 2>/dev/null
