#!/bin/bash
# usage: tools/multi_r2.sh N -- dist parity + weak bench (device loop) + weak bench (python loop)
N=$1
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) tools/dist_parity.py > gpurun_out/dp_$N.log 2>&1; echo "parity rc=$?"; grep -E "^(OK|BAD)" gpurun_out/dp_$N.log | sort | uniq -c | sort -rn | head -20
for dl in 1 0; do
PMSZ_DEVLOOP=$dl timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
   --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-cpu-baseline --no-e2e > gpurun_out/w_${N}_$dl.log 2>&1
echo "devloop=$dl rc=$?"; grep '^{' gpurun_out/w_${N}_$dl.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('  ', round(d['ms_per_step'],3), '%.3e'%d['value'], 'rounds', d['result']['rounds'], 'syncs', d['result']['syncs'], d['result']['edits_per_round'], 'iters', [r['iterations'] for r in d['result']['per_rank']])"
done
