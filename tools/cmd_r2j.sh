mkdir -p gpurun_out; timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > gpurun_out/gputests_r2j.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_r2j.log
timeout 300 python bench.py --no-cpu-baseline --no-dropin > gpurun_out/b_r2j.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-dropin --f64-original > gpurun_out/b64j.json 2>&1
for f in b_r2j b64j; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['ms_per_step'],3), {k:round(v['ms_total_per_step'],3) for k,v in d['roofline']['per_kernel'].items()}, d['e2e']['ms_per_step'], d['result']['reference_pin']['bit_exact'], d['result']['residual'], d['result']['fragile_fraction'])"; done
