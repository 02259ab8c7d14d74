#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -2
for lib in libpmsz.so libpmsz_old.so libpmsz.so libpmsz_old.so; do
PMSZ_LIB=paper_2601_01787_b200/_lib/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-dropin > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']; print('$lib', round(d['ms_per_step'],3), 'prep', round(pk['prep']['ms_per_launch'],4), d['result'].get('reference_pin',{}).get('bit_exact'))"
done
PMSZ_LIB=paper_2601_01787_b200/_lib/libpmsz.so timeout 600 python bench.py --f64-original --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-dropin > /tmp/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']; print('f64 new', round(d['ms_per_step'],3), 'prep', round(pk['prep']['ms_per_launch'],4), d['result'].get('reference_pin',{}).get('bit_exact'))"
