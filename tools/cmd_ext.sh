#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --workload hedm --no-cpu-baseline --no-dropin --no-e2e > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']
print('hedm', round(d['ms_per_step'],3), 'fragile', d['result'].get('fragile_fraction'), {k: round(v['ms_total_per_step'],3) for k,v in pk.items()}, d['result']['edits_per_iteration'][:6])"
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --no-e2e > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('default', round(d['ms_per_step'],3), d['result'].get('reference_pin',{}).get('bit_exact'))"
