#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --no-e2e > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']; print('$*', round(d['ms_per_step'],3), 'tail', round(pk['tail']['ms_total_per_step'],3))"; }
run X=0
run PMSZ_TAIL_PER_SM=2
run PMSZ_TAIL_BLOCKS=74
run PMSZ_TAIL_BLOCKS=37
run X=0
