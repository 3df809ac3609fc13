set -u
O=gpurun_out/r2l; mkdir -p $O
for r in 1 2; do for L in paper_1802_01359_b200/libfif_b200.so variants/nopark.so; do
  FIF_LIB_PATH=$L timeout 300 python tools/run_plan.py --config cfg2 --batch 512 --reps 4 2>&1 | tail -1 | sed "s|^|$L |"
done; done 2>&1 | tee $O/ab.txt
