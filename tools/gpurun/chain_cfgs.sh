#!/bin/bash
# chain timings (forward + backward variants) per config and gemm knob settings
mkdir -p gpurun_out
tag=${1:-a}
for cfg in ${CFGS:-products reddit}; do
for st in ${SETTINGS:-default}; do
  env $( [ "$st" != default ] && echo $st ) timeout 1200 python bench.py --config $cfg --no-cpu --no-e2e --steps 10 > gpurun_out/chain_${cfg}_${tag}.json 2> gpurun_out/chain_${cfg}_${tag}.log
  python -c "
import json;d=json.load(open('gpurun_out/chain_${cfg}_${tag}.json'));c=d['chain'];print('$cfg', '$st', d['ms_per_step'], {k: c[k] for k in ('forward_ms','backward_epp_ms','backward_epp_global_ms','backward_all_active_ms','backward_ifelse_ms','backward_epp_tensor_core_ms')})"
done
done
