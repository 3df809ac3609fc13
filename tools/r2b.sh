set -u
O=gpurun_out/m; mkdir -p $O
bash tools/profile_one.sh full1
ncu -i $O/full_resident.ncu-rep --page raw --csv > $O/full_resident_raw.csv 2>/dev/null
ncu -i $O/full_resident.ncu-rep --page source --csv --print-source sass > $O/full_resident_src.csv 2>/dev/null
ls -la $O
