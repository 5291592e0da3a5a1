#!/bin/bash
mkdir -p gpurun_out
PG_BENCH_FORCE_COMM=1 timeout 600 python bench.py --no-chain --no-cpu --no-e2e --steps 5 > gpurun_out/r2_forcecomm.json 2> gpurun_out/r2_forcecomm.log
echo "force-comm rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/r2_forcecomm.json').read().strip().splitlines()[-1]);print('force comm', d['ms_per_step'], d['parity'])"
PG_BENCH_BACKEND=gloo PG_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/r2_rehearsal2.json 2> gpurun_out/r2_rehearsal2.log
echo "rehearsal rc=$?"; tail -c 1500 gpurun_out/r2_rehearsal2.json; grep -iE "error|Traceback" gpurun_out/r2_rehearsal2.log | head -5
