#!/bin/bash
# whole-row SpMM warps (k_agg_row): parity tests with the knob on, then a knob sweep on the reddit shape
mkdir -p gpurun_out
tag=${1:-a}
PG_ROW_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_fullsize.py -x -q > gpurun_out/row_pytest_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/row_pytest_$tag.log
DEF='[{}, {"row_kernel":1}]'
PG_BENCH_SWEEP=${SWEEP:-$DEF} \
  timeout 1200 python bench.py --no-chain --no-cpu --no-e2e --steps 5 > gpurun_out/row_sweep_$tag.json 2> gpurun_out/row_sweep_$tag.log
echo "bench rc=$?"; grep "\[sweep\]" gpurun_out/row_sweep_$tag.log
