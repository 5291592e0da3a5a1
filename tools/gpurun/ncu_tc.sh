#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_abt_tc -s 1 -c 1 -f -o gpurun_out/r2_ncu_abt \
  python tools/prof_gemm_tc.py --ncu --only=products\ layer0\ y > gpurun_out/r2_ncu_abt.log 2>&1
echo "abt rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gemm_atb_tc -s 1 -c 1 -f -o gpurun_out/r2_ncu_atb \
  python -c "import sys; sys.argv=['x','--only=products layer0 W']; sys.path.insert(0,'tools'); import prof_gemm_tc as p; p.main_atb()" > gpurun_out/r2_ncu_atb.log 2>&1
echo "atb rc=$?"
