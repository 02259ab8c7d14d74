#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 1 0 1 0; do
PMSZ_HOST_FILL=$v PMSZ_E2E_TRACE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-dropin > /tmp/b.json 2> /tmp/b.err
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('host_fill=$v e2e', round(d['e2e']['ms_per_step'],2), d['e2e']['check'])"
grep "e2e:" /tmp/b.err | tail -2
done
