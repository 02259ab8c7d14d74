mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_v36.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gputests_v36.log
python bench.py > gpurun_out/bench_v36_default.json 2>gpurun_out/bench_v36.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_v36_default.json')); print(d['ms_per_step'], d['roofline']['frac'], {k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()})"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 > gpurun_out/bench_v36_2gpu.log 2>&1; echo multi rc=$?
grep '^{' gpurun_out/bench_v36_2gpu.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], {k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()})"
