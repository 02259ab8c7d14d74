# Weak-scaling bench lines only (perlin 512^3 per GPU) at N = 4 and 2 (run under gpurun --gpus 4)
for N in 4 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
     --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $N > gpurun_out/weak_$N.log 2>&1
  echo "N=$N rc=$?"; grep '^{' gpurun_out/weak_$N.log > gpurun_out/weak_$N.json
  python -c "import json; d=json.load(open('gpurun_out/weak_$N.json')); print($N, d['ms_per_step'], '%.4g' % d['value'])"
done
