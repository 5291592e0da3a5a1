#!/bin/bash
# randomised soak: stage / host pipeline / build / tolerance kernels with many seeds
mkdir -p gpurun_out
PG_STRESS_SEEDS=${1:-400} PG_STRESS_SEEDS_TOL=${2:-200} timeout 3000 python -m pytest tests/test_gpu_stress.py -q -x -p no:cacheprovider > gpurun_out/r2_soak.log 2>&1
echo "soak rc=$?"; tail -5 gpurun_out/r2_soak.log
