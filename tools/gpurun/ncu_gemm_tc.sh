#!/bin/bash
# ncu --set full of the tensor-core gemm_a_bt at the products layer-0 shape
mkdir -p gpurun_out
timeout 300 python tools/prof_gemm_tc.py > gpurun_out/r2_gemm_tc_prof.log 2>&1
cat gpurun_out/r2_gemm_tc_prof.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_abt_tc -s 1 -c 1 \
  -o gpurun_out/r2_ncu_gemm_tc -f python tools/prof_gemm_tc.py --ncu --only=products > gpurun_out/r2_ncu_gemm_tc.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2_ncu_gemm_tc.log
