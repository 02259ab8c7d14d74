mkdir -p gpurun_out; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_parallel_api.py -m gpu -x -q > gpurun_out/gputests_r2l.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_r2l.log
timeout 300 python bench.py --no-cpu-baseline --no-dropin --no-e2e > gpurun_out/b_r2l.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/b_r2l.json')); print(round(d['ms_per_step'],3), {k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()}, d['result']['reference_pin']['bit_exact'], d['result']['residual'])"
PMSZ_TAIL_TRACE=1 timeout 300 python tools/one_run.py 512 1 2>&1 | grep -A1 "tail"
