# GPU tests (incl. the multi-GPU parity tests) and two 2-GPU bench lines (run under gpurun --gpus 2)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_chk.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gputests_chk.log
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 2 --no-e2e > gpurun_out/chk_2gpu.log 2>&1; echo multi rc=$?
grep '^{' gpurun_out/chk_2gpu.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['result']; print(d['ms_per_step'], d['value'], r['rounds'], r['syncs'], r['edits_per_round'], r['residual'])"
done
