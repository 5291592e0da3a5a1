#!/bin/bash
mkdir -p gpurun_out
PG_REC_WINDOW=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg -f -o gpurun_out/r2_ncu_reddit_rw \
   python bench.py --config reddit --profile --ncu-path > gpurun_out/r2_ncu_reddit_rw.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2_ncu_reddit_rw.ncu-rep --page raw --csv > gpurun_out/r2_ncu_reddit_rw_raw.csv 2>/dev/null
