#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/multi_r2.sh 2
for v in 1 0; do
PMSZ_PDL=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('pdl=$v', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), d['result'].get('reference_pin',{}).get('bit_exact'))"
done
