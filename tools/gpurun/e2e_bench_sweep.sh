#!/bin/bash
# host-pipeline knob sweep inside bench.py's own e2e measurement (PG_BENCH_E2E_SWEEP)
mkdir -p gpurun_out
tag=${1:-a}
PG_BENCH_E2E_SWEEP="$SWEEP" timeout 1200 python bench.py --no-chain --no-cpu --steps 5 > gpurun_out/e2e_bsweep_$tag.json 2> gpurun_out/e2e_bsweep_$tag.log
echo "bench rc=$?"; grep -E "e2e-sweep|\[e2e\]" gpurun_out/e2e_bsweep_$tag.log
