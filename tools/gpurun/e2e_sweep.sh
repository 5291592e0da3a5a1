#!/bin/bash
# host-pipeline knob sweep of the e2e epoch (pinned, then pageable)
mkdir -p gpurun_out
tag=${1:-a}
DEF='[{}]'
S1=${SWEEP:-$DEF}
S2=${SWEEP2:-$DEF}
timeout 900 python tools/sweep_e2e.py "$S1" pinned > gpurun_out/e2e_sweep_$tag.log 2>&1
echo "pinned rc=$?"; grep "\[e2e" gpurun_out/e2e_sweep_$tag.log
timeout 900 python tools/sweep_e2e.py "$S2" pageable > gpurun_out/e2e_sweep_pg_$tag.log 2>&1
echo "pageable rc=$?"; grep "\[e2e" gpurun_out/e2e_sweep_pg_$tag.log
