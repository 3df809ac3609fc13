# A/B timing of alternative builds on the mixed-radix fp32 config-4 lengths (dev tool)
for r in 1 2; do for L in "$@"; do
  echo "$L 3*2^14 $(FIF_LIB_PATH=$L python tools/run_plan.py --config cfg4 --n 49152 --batch 5461 --reps 3 | tail -1 | cut -c1-20) 5*2^14 $(FIF_LIB_PATH=$L python tools/run_plan.py --config cfg4 --n 81920 --batch 3276 --reps 3 | tail -1 | cut -c1-20)"
done; done
