#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_gpu_aggregate.py -x -q > gpurun_out/r2_grouped_pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r2_grouped_pytest.log
timeout 600 python tools/prof_grouped.py reddit > gpurun_out/r2_grouped_prof_reddit.log 2>&1
timeout 300 python tools/prof_grouped.py arxiv > gpurun_out/r2_grouped_prof_arxiv.log 2>&1
cat gpurun_out/r2_grouped_prof_reddit.log gpurun_out/r2_grouped_prof_arxiv.log
