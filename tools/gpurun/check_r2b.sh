#!/bin/bash
# session re-entry check: gpu suite + smoke, default bench, one ncu capture of the reddit layer-0 path (raw csv)
mkdir -p gpurun_out
bash tools/gpurun/full_gpu_suite.sh
timeout 1200 python bench.py > gpurun_out/bench_r02_b.json 2> gpurun_out/bench_r02_b.log
echo "bench rc=$?"; tail -c 400 gpurun_out/bench_r02_b.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg -f -o gpurun_out/r2b_ncu_reddit \
   python bench.py --config reddit --profile --ncu-path > gpurun_out/r2b_ncu_reddit.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2b_ncu_reddit.ncu-rep --page raw --csv > gpurun_out/r2b_ncu_reddit_raw.csv 2>/dev/null
ls -la gpurun_out
