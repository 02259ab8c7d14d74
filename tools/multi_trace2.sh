#!/bin/bash
N=$1; shift
PMSZ_DIST_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-cpu-baseline --no-e2e --steps 5 "$@" > gpurun_out/mt2_${N}.log 2>&1
grep '^{' gpurun_out/mt2_${N}.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d['ms_per_step'],3))
    for r in d['result']['per_rank']: print(r['rank'], r['iterations'], r['trace_ms_per_step'])"
