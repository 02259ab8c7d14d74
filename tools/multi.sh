#!/bin/bash
# usage: tools/multi.sh N [extra bench args...]  -- one torchrun bench line per workload
N=$1; shift
for wl in perlin hedm strong; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --workload $wl "$@" \
     > gpurun_out/multi_${N}_${wl}.log 2>&1
  echo "$wl rc=$?"; grep '^{' gpurun_out/multi_${N}_${wl}.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'], d['ms_per_step'], '%.3e'%d['value'], d.get('e2e',{}).get('value'), d['result']['rounds'], d['result']['syncs'])"
done
