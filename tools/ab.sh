# A/B timing of alternative builds (dev tool): bash tools/ab.sh lib1.so lib2.so ...
for L in "$@"; do
  echo "== $L"
  FIF_LIB_PATH=$L python tools/run_plan.py --config cfg4 --n 131072 --batch 2048 --reps 3 | tail -1
  FIF_LIB_PATH=$L python tools/run_plan.py --config cfg2 --reps 3 | tail -1
  FIF_LIB_PATH=$L python tools/run_plan.py --config cfg3 --reps 3 | tail -1
done
