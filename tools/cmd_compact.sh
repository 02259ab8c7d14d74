#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c.log 2>&1 || { tail -20 gpurun_out/build_c.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests_c.log 2>&1
echo tests=$?; tail -2 gpurun_out/gputests_c.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-dropin > gpurun_out/b_c$i.json 2> gpurun_out/b_c.err
python -c "
import json; d=json.loads(open('gpurun_out/b_c$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['result'].get('reference_pin',{}).get('bit_exact'))"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dropin > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv
from collections import defaultdict
rows = list(csv.reader(open('gpurun_out/launches_c.csv')))
hi = next(i for i,r in enumerate(rows) if r and r[0]=='ID')
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
seq = [(r[ki], float(r[vi])) for r in rows[hi+1:] if len(r) > vi]
idx = [i for i,(k,v) in enumerate(seq) if 'k_prep_q' in k]
agg = defaultdict(lambda: [0,0.0])
for k, v in seq[idx[-1]:]:
    n = k.split('(')[0].replace('void ',''); agg[n][0]+=1; agg[n][1]+=v/1000
for n,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{n[:50]:50s} {c:3d} {t:8.1f} us")
P
