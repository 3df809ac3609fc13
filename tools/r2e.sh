set -u
O=gpurun_out/r2e; mkdir -p $O
bash tools/ab_res.sh variants/old.so paper_1802_01359_b200/libfif_b200.so variants/ltab.so 2>&1 | tee $O/ab.txt
