# A/B timing of alternative builds on the fp64 streamed configs (dev tool)
for r in 1 2; do for L in "$@"; do
  echo "$L cfg2 $(FIF_LIB_PATH=$L python tools/run_plan.py --config cfg2 --reps 3 | tail -1 | cut -c1-20) cfg3 $(FIF_LIB_PATH=$L python tools/run_plan.py --config cfg3 --reps 3 | tail -1 | cut -c1-20)"
done; done
