#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --no-e2e > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],3))"; }
run X=0
run PMSZ_TAIL1_MAX=1024
run PMSZ_TAIL1_MAX=256
run PMSZ_DENSE_MIN=262144
run PMSZ_DENSE_MIN=1048576
run PMSZ_DEFER_PER_SM=4
run PMSZ_APPLY_PER_SM=2
run PMSZ_PREP_ZCHUNK=32
run X=0
