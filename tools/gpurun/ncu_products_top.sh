#!/bin/bash
# ncu --set full of the products top path (dim 256): the launches of path 0 of one bench step
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_agg" -c 3 -f -o gpurun_out/r2_ncu_ptop \
   python bench.py --config products --profile --steps 1 --warmup 1 --no-chain --no-e2e --no-cpu > gpurun_out/r2_ncu_ptop.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2_ncu_ptop.ncu-rep --page raw --csv > gpurun_out/r2_ncu_ptop_raw.csv 2>/dev/null
rm -f gpurun_out/r2_ncu_ptop.ncu-rep
