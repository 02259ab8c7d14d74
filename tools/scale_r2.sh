#!/bin/bash
# usage: tools/scale_r2.sh N -- weak (tile) + strong slab + strong block + hedm lines at N GPUs
N=$1; shift
mkdir -p gpurun_out
run() {
  tag=$1; shift
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-cpu-baseline "$@" > gpurun_out/s_${N}_${tag}.log 2>&1
  echo "$tag N=$N rc=$?"; grep '^{' gpurun_out/s_${N}_${tag}.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  ', round(d['ms_per_step'],3), '%.3e'%d['value'], 'e2e', d.get('e2e',{}).get('ms_per_step'), 'rounds', d['result']['rounds'], 'syncs', d['result']['syncs'], 'iters', [r['iterations'] for r in d['result']['per_rank']], 'edits', [r['edits'] for r in d['result']['per_rank']])"
}
run weak
run strong_slab --workload strong
run strong_block --workload strong --decomp block
run hedm --workload hedm
