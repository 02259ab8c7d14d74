#!/bin/bash
# usage: tools/multi_trace.sh N [extra bench args]  -- weak scaling line + a traced run
N=$1; shift
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-cpu-baseline --no-e2e "$@" > gpurun_out/mt_${N}.log 2>&1
echo "N=$N rc=$?"
PMSZ_DIST_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-cpu-baseline --no-e2e --steps 3 "$@" > gpurun_out/mt_${N}_trace.log 2>&1
for f in gpurun_out/mt_${N}.log gpurun_out/mt_${N}_trace.log; do grep '^{' $f | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(round(d['ms_per_step'],3), '%.3e'%d['value'], 'rounds', d['result']['rounds'], d['result']['edits_per_round'], 'iters', [r['iterations'] for r in d['result']['per_rank']], 'edits', [r['edits'] for r in d['result']['per_rank']], 'ms', [round(r['ms'],3) for r in d['result']['per_rank']]); print(d.get('trace_ms_per_step'))"; done
