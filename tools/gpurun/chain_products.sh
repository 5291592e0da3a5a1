#!/bin/bash
mkdir -p gpurun_out
tag=${1:-a}
for gp in ${GP:-2 1}; do
  PG_GEMM_PACKED=$gp timeout 1200 python bench.py --config products --no-cpu --no-e2e --steps 10 > gpurun_out/chain_products_${tag}_$gp.json 2> gpurun_out/chain_products_${tag}_$gp.log
  python -c "
import json;d=json.load(open('gpurun_out/chain_products_${tag}_$gp.json'));c=d['chain'];print('gemm_packed=$gp', d['ms_per_step'], {k: c[k] for k in ('forward_ms','backward_epp_ms','backward_epp_global_ms','backward_all_active_ms','backward_ifelse_ms','backward_epp_tensor_core_ms')})"
done
