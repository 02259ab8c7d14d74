#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in 1 0 1 0; do
PMSZ_SYNC_KERNEL=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('sync_kernel=$v', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), 'dropin', round(d['dropin']['ms_per_call'],1))"
done
