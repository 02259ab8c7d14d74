# Multi-GPU bench lines for every workload (run under gpurun --gpus N): bash tools/scale_round.sh N
N=$1
bash tools/multi.sh $N
for wl in perlin hedm strong; do grep '^{' gpurun_out/multi_${N}_${wl}.log; done > gpurun_out/scale_$N.jsonl
