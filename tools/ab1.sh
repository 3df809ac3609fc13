# A/B timing of alternative builds on config 1 (dev tool): bash tools/ab1.sh lib1.so lib2.so ...
for r in 1 2; do for L in "$@"; do
  echo "$L $(FIF_LIB_PATH=$L python tools/run_plan.py --config cfg1 --reps 6 --eig | tail -1 | cut -c1-20)"
done; done
