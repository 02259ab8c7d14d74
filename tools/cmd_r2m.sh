mkdir -p gpurun_out; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_parallel_api.py tests/test_integration_stub.py -m gpu -x -q > gpurun_out/gputests_r2m.log 2>&1; echo tests=$?; tail -3 gpurun_out/gputests_r2m.log
for cfg in "PMSZ_RULES1=0" "PMSZ_RULES1=1"; do
env $cfg timeout 300 python bench.py --no-cpu-baseline --no-dropin --no-e2e > gpurun_out/b_r2m.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/b_r2m.json')); print('$cfg', round(d['ms_per_step'],3), {k:(round(v['ms_total_per_step'],3), v['launches_per_step']) for k,v in d['roofline']['per_kernel'].items()}, d['result']['reference_pin']['bit_exact'], d['result']['residual'])"
done
