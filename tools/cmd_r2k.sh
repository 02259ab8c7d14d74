mkdir -p gpurun_out; timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r2k.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_r2k.log
PMSZ_E2E_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-dropin --steps 3 2>&1 | grep -E "e2e:" | tail -2
timeout 600 python bench.py > gpurun_out/b_r2k.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/b_r2k.json')); print(round(d['ms_per_step'],3), {k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()}, d['e2e']['ms_per_step'], d['dropin']['ms_per_call'], d['result']['reference_pin']['bit_exact'], d['result']['residual'], d['gpu_launches']/d['steps'])"
