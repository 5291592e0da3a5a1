#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stress.py -x -q -k "stage or host_pipeline" > gpurun_out/r2_stress.log 2>&1
echo "stress rc=$?"; tail -2 gpurun_out/r2_stress.log
for rw in 1 0 1; do
  PG_REC_WINDOW=$rw timeout 600 python bench.py --no-chain --no-cpu --no-e2e --steps 20 > gpurun_out/r2_perf_rw$rw.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2_perf_rw$rw.json').read().strip().splitlines()[-1]);print('rec_window=$rw', d['ms_per_step'], d['per_path_ms'], d['parity']['all'])"
done
for nt in 1 0; do
  PG_STAGE_NT=$nt timeout 600 python bench.py --no-chain --no-cpu --steps 5 > gpurun_out/r2_perf_nt$nt.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r2_perf_nt$nt.json').read().strip().splitlines()[-1]);e=d['e2e'];print('stage_nt=$nt e2e', e['ms_per_step'], 'pageable', e['pageable_ms_per_step'])"
done
