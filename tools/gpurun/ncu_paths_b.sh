#!/bin/bash
# ncu --set full of one execution of each config's dominant path + the launch list of a short bench
mkdir -p gpurun_out
tag=${1:-b}
for cfg in reddit products arxiv; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_agg -f -o gpurun_out/r2${tag}_ncu_$cfg \
     python bench.py --config $cfg --profile --ncu-path > gpurun_out/r2${tag}_ncu_$cfg.log 2>&1
  echo "$cfg ncu rc=$?"; grep "ncu-path" gpurun_out/r2${tag}_ncu_$cfg.log
  ncu -i gpurun_out/r2${tag}_ncu_$cfg.ncu-rep --page raw --csv > gpurun_out/r2${tag}_ncu_${cfg}_raw.csv 2>/dev/null
  rm -f gpurun_out/r2${tag}_ncu_$cfg.ncu-rep
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2${tag}_launches.csv \
   python bench.py --profile --steps 2 --warmup 1 > gpurun_out/r2${tag}_launches_bench.log 2>&1
echo "launches rc=$?"
