#!/bin/bash
# GPU-box session: tensor-core gemm_a_bt tests + timing (+ ncu of one launch)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm_tc.py -x -q > gpurun_out/r2_gemm_tc_pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r2_gemm_tc_pytest.log
timeout 300 python tools/prof_gemm_tc.py > gpurun_out/r2_gemm_tc_prof.log 2>&1
echo "prof rc=$?"; cat gpurun_out/r2_gemm_tc_prof.log
