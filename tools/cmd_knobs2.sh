#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --no-e2e > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],3), d['result'].get('reference_pin',{}).get('bit_exact'))"; }
run X=0
run PMSZ_QMASK=1
run PMSZ_FULL_DIV=4
run PMSZ_FULL_DIV=16
run PMSZ_SORT_MIN=131072
run PMSZ_SORT_MIN=524288
run X=0
