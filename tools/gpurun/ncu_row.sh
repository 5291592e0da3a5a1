#!/bin/bash
# ncu --set full of one reddit layer-0 path execution with the whole-row kernel
mkdir -p gpurun_out
tag=${1:-a}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg -f -o gpurun_out/row_ncu_$tag \
   python bench.py --config reddit --profile --ncu-path > gpurun_out/row_ncu_$tag.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/row_ncu_$tag.ncu-rep --page raw --csv > gpurun_out/row_ncu_${tag}_raw.csv 2>/dev/null
ls -la gpurun_out/row_ncu_$tag*
