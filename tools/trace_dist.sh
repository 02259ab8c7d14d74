# Round-phase breakdown of the relaxed multi-GPU loop (PMSZ_DIST_TRACE=1 synchronises every phase)
N=${1:-2}
PMSZ_DIST_TRACE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N --no-e2e --no-cpu-baseline > gpurun_out/trace_$N.log 2>&1
grep 'trace_ms' gpurun_out/trace_$N.log | head -1 > /dev/null
grep '^{' gpurun_out/trace_$N.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ms_per_step'], d['trace_ms_per_step']); print({k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()}); print([(r['rank'], r['iterations']) for r in d['result']['per_rank']], d['result']['edits_per_round'])"
