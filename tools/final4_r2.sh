#!/bin/bash
# Round-2 final multi-GPU set on N GPUs: multi-GPU tests, dist parity, weak (device + python loop), strong, hedm, reference arm.
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu > gpurun_out/gputests_multi_$N.log 2>&1; echo multitests rc=$?; tail -2 gpurun_out/gputests_multi_$N.log
bash tools/multi_r2.sh $N
bash tools/scale_r2.sh $N 2>&1 | grep -v "^weak"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) \
   bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/ref_$N.log 2>&1; echo "reference rc=$?"; grep '^{' gpurun_out/ref_$N.log | cut -c1-200
