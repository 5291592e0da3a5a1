#!/bin/bash
# 256-bit row gathers (k_agg_vec8): parity with the knob on, then per-path sweeps on the configs
mkdir -p gpurun_out
tag=${1:-a}
PG_VEC8=1 timeout 900 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullsize.py -x -q > gpurun_out/vec8_pytest_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/vec8_pytest_$tag.log
DEF='[{}, {"vec8":1}, {}, {"vec8":1}]'
for cfg in ${CONFIGS:-reddit products arxiv}; do
PG_BENCH_SWEEP=${SWEEP:-$DEF} \
  timeout 1200 python bench.py --config $cfg --no-chain --no-cpu --no-e2e --steps 5 > gpurun_out/vec8_sweep_${cfg}_$tag.json 2> gpurun_out/vec8_sweep_${cfg}_$tag.log
echo "bench $cfg rc=$?"; grep "\[sweep\]" gpurun_out/vec8_sweep_${cfg}_$tag.log
done
