#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_f64.py tests/test_gpu_gemm_tc.py -q -x --tb=short 2>&1 | tail -30
