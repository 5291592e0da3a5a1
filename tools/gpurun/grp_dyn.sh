#!/bin/bash
# grouped Fast: dynamic group hand-out (grp_dynamic) parity + timing per gs
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py -x -q > gpurun_out/grp_dyn_pytest.log 2>&1
echo "pytest rc=$?"; tail -1 gpurun_out/grp_dyn_pytest.log
for d in 0 1; do PG_GRP_DYNAMIC=$d timeout 900 python tools/prof_grouped.py reddit 42 61 128 2>&1 | grep -v "^\s*$" | sed "s/^/dyn=$d /"; done
