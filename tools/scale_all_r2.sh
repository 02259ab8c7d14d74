#!/bin/bash
# N = 1 anchors + N = 2 and 4 lines of every workload on one 4-GPU box (tools/scale_r2.sh)
mkdir -p gpurun_out
for wl in default strong hedm; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --no-dropin --no-e2e > gpurun_out/s_1_$wl.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/s_1_$wl.json').read().strip().splitlines()[-1]); print('$wl N=1', round(d['ms_per_step'],3), '%.3e'%d['value'])"
done
bash tools/scale_r2.sh 2
bash tools/scale_r2.sh 4
