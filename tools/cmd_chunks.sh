#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c.log 2>&1 || { tail -20 gpurun_out/build_c.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/gputests_c.log 2>&1
echo tests=$?; tail -2 gpurun_out/gputests_c.log
for ps in 6 16 27 6 16 27; do
PMSZ_COMPACT_PER_SM=$ps timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-dropin > gpurun_out/b_ch.json 2> gpurun_out/b_ch.err
python -c "
import json; d=json.loads(open('gpurun_out/b_ch.json').read().strip().splitlines()[-1]); pk=d['roofline']['per_kernel']; print('per_sm=$ps', round(d['ms_per_step'],3), 'compact', round(pk['compact']['ms_total_per_step'],3), d['result'].get('reference_pin',{}).get('bit_exact'))"
done
