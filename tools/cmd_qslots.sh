#!/bin/bash
for lib in libpmsz.so libpmsz_q8_2.so libpmsz_q4_4.so libpmsz_q5_3.so libpmsz_q7_2.so libpmsz.so; do
PMSZ_LIB=paper_2601_01787_b200/_lib/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-dropin > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']; print('$lib', round(d['ms_per_step'],3), 'sweep_full', round(pk['sweep_full']['ms_per_launch'],3), d['result'].get('reference_pin',{}).get('bit_exact'))"
done
