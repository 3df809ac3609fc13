set -u
O=gpurun_out/r2f; mkdir -p $O
python tools/run_plan.py --config cfg2 --batch 512 --reps 2 > $O/plain_cl.log 2>&1; cat $O/plain_cl.log
ncu --set full --clock-control none --import-source on -k regex:fif_cluster_kernel -s 1 -c 1 -o $O/full_cluster \
  python tools/run_plan.py --config cfg2 --batch 512 --reps 2 > $O/ncu_cl.log 2>&1; echo "ncu1 rc=$?"
ncu -i $O/full_cluster.ncu-rep --page raw --csv > $O/full_cluster_raw.csv 2>/dev/null
ncu -i $O/full_cluster.ncu-rep --page source --csv --print-source sass > $O/full_cluster_src.csv 2>/dev/null
python tools/run_plan.py --config cfg4 --n 131072 --batch 2048 --reps 2 > $O/plain_st.log 2>&1; cat $O/plain_st.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -s 40 -c 60 --log-file $O/launches_cfg4_131072.csv python tools/run_plan.py --config cfg4 --n 131072 --batch 2048 --reps 2 > $O/ncu_st.log 2>&1; echo "ncu2 rc=$?"
ls -la $O
