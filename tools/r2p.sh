set -u
O=gpurun_out/r2p; mkdir -p $O
bash tools/ab_res.sh paper_1802_01359_b200/libfif_b200.so variants/hk8.so variants/hk16.so 2>&1 | tee $O/ab.txt
