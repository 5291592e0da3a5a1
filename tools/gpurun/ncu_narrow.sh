#!/bin/bash
# ncu --set full of the Reddit top path (dim 16): the narrow main kernel and the concurrent hub kernel
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:k_agg_vec4<.int.4,|k_agg_heavy_coop" -c 4 -f -o gpurun_out/r2_ncu_narrow \
   python bench.py --config reddit --profile --steps 1 --warmup 1 --no-chain --no-e2e --no-cpu > gpurun_out/r2_ncu_narrow.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2_ncu_narrow.ncu-rep --page raw --csv > gpurun_out/r2_ncu_narrow_raw.csv 2>/dev/null
rm -f gpurun_out/r2_ncu_narrow.ncu-rep
