#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ep.log 2>&1 || { tail -20 gpurun_out/build_ep.log; exit 1; }
timeout 900 python -m pytest tests/test_integration_stub.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gputests_ep.log 2>&1
echo tests=$?; tail -2 gpurun_out/gputests_ep.log
for v in 1 0 1 0; do
PMSZ_EARLY_PATCH=$v PMSZ_E2E_TRACE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b_ep$v.json 2> gpurun_out/b_ep$v.err
python -c "
import json; d=json.loads(open('gpurun_out/b_ep$v.json').read().strip().splitlines()[-1]); print('ep=$v', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['check'], 'dropin', round(d['dropin']['ms_per_call'],1), d['dropin']['matches_device'])"
grep "e2e:" gpurun_out/b_ep$v.err | tail -2
done
