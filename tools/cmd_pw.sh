#!/bin/bash
# host patch: prefetchw build (libpmsz_pw.so) vs the default build, e2e and drop-in legs
mkdir -p gpurun_out
for lib in paper_2601_01787_b200/_lib/libpmsz_pw.so paper_2601_01787_b200/_lib/libpmsz.so paper_2601_01787_b200/_lib/libpmsz_pw.so paper_2601_01787_b200/_lib/libpmsz.so; do
PMSZ_LIB=$lib PMSZ_E2E_TRACE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/b_pw.json 2> gpurun_out/b_pw.err
python -c "
import json; d=json.loads(open('gpurun_out/b_pw.json').read().strip().splitlines()[-1]); print('$lib'.split('/')[-1], round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2), 'dropin', round(d['dropin']['ms_per_call'],1))"
grep "e2e:" gpurun_out/b_pw.err | tail -2
done
