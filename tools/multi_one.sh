#!/bin/bash
# usage: tools/multi_one.sh N workload [extra bench args...]
N=$1; wl=$2; shift 2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --workload $wl "$@" > gpurun_out/m_${N}_${wl}.log 2>&1
echo "$wl N=$N rc=$?"; grep '^{' gpurun_out/m_${N}_${wl}.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], '%.3e'%d['value'], d['result']['rounds'], d['result']['edits_per_round'], [r['iterations'] for r in d['result']['per_rank']])"
