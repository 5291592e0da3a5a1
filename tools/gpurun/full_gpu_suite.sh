#!/bin/bash
# the whole -m gpu suite, then smoke()
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/r2_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?"; tail -3 gpurun_out/r2_smoke.log
