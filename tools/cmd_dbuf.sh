#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_db.log 2>&1 || { tail -20 gpurun_out/build_db.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests_db.log 2>&1
echo tests=$?; tail -3 gpurun_out/gputests_db.log
for v in 1 0 1 0; do
PMSZ_DEFER_BUF=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-dropin > gpurun_out/b_db$v.json 2> gpurun_out/b_db$v.err
python - <<P
import json
d=json.loads(open('gpurun_out/b_db$v.json').read().strip().splitlines()[-1])
pk=d['roofline'].get('per_kernel',{})
print('buf=$v', round(d['ms_per_step'],3), {k: round(v,3) if isinstance(v,float) else v for k,v in pk.items()} if pk else '', d['result'].get('reference_pin',{}).get('bit_exact'))
P
done
