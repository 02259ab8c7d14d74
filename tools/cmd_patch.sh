#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_integration_stub.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2 3; do
PMSZ_E2E_TRACE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /tmp/b.json 2> /tmp/b.err
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['check'], 'dropin', round(d['dropin']['ms_per_call'],1))"
grep "e2e:" /tmp/b.err | sed -n '4,5p'
done
