#!/bin/bash
# GPU-box session: full-size parity tests + the default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_stress.py::test_concurrent_calls_share_one_grouping tests/test_capi.py -x -q --durations=10 > gpurun_out/r2_pytest_fullsize.log 2>&1
echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_a.json 2> gpurun_out/r2_bench_a.err
echo "bench rc=$?"
tail -3 gpurun_out/r2_pytest_fullsize.log
