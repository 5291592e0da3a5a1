#!/bin/bash
mkdir -p gpurun_out
for cfg in products reddit; do
  timeout 900 python bench.py --config $cfg --no-cpu --no-e2e --steps 5 > gpurun_out/r2_chain_$cfg.json 2> gpurun_out/r2_chain_$cfg.log
  python -c "import json;d=json.loads(open('gpurun_out/r2_chain_$cfg.json').read().strip().splitlines()[-1]);c=d['chain'];print('$cfg', {k:v for k,v in c.items() if 'ms' in k or 'err' in k})"
done
PG_HOST_TRACE=1 timeout 900 python bench.py --no-cpu --no-chain --steps 3 > gpurun_out/r2_trace.json 2> gpurun_out/r2_trace.log
grep host_trace gpurun_out/r2_trace.log | tail -6
