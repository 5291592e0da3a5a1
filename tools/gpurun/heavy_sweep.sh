#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --heavy-sweep --no-chain --no-cpu --no-e2e --steps 10 > gpurun_out/r2_heavy_sweep.json 2> gpurun_out/r2_heavy_sweep.err
echo "rc=$?"; grep -E "\[sweep\]|\[shards\]|\[segments\]" gpurun_out/r2_heavy_sweep.err | head -40
