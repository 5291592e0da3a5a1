#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm_tc.py -x -q > gpurun_out/r2_gemm_tc_pytest.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/r2_gemm_tc_pytest.log
timeout 600 python tools/prof_gemm_tc.py > gpurun_out/r2_gemm_tc_prof2.log 2>&1
echo "prof rc=$?"; cat gpurun_out/r2_gemm_tc_prof2.log
PG_GEMM_TC=1 timeout 900 python bench.py --config products --no-cpu --no-e2e --steps 5 > gpurun_out/r2_products_tc.json 2> gpurun_out/r2_products_tc.log
python -c "import json;d=json.loads(open('gpurun_out/r2_products_tc.json').read().strip().splitlines()[-1]);print('products chain with gemm_tc=1', d['chain'])"
