#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_di.log 2>&1 || { tail -20 gpurun_out/build_di.log; exit 1; }
timeout 900 python -m pytest tests/test_integration_stub.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gputests_di.log 2>&1
echo tests=$?; tail -5 gpurun_out/gputests_di.log
timeout 300 python tools/dropin_timing.py 2>&1 | head -3
PMSZ_E2E_TRACE=1 timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b_di.json 2> gpurun_out/b_di.err
echo bench=$?
python - <<'P'
import json
d=json.loads(open('gpurun_out/b_di.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['value'], d.get('dropin',{}).get('ms_per_call'), d.get('dropin',{}).get('matches_device'))
P
grep "e2e:" gpurun_out/b_di.err | tail -8
