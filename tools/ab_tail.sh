mkdir -p gpurun_out
for cfg in "PMSZ_X=0" "PMSZ_DENSE_MIN=262144" "PMSZ_DENSE_MIN=524288" "PMSZ_TAIL_PER_SM=2" "PMSZ_TAIL_PER_SM=2 PMSZ_DENSE_MIN=524288" "PMSZ_TAIL1_MAX=1024" "PMSZ_TAIL1_MAX=256"; do
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-dropin --steps 10 > gpurun_out/ab.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$cfg', round(d['ms_per_step'],3), {k:(round(v['ms_total_per_step'],3), v['launches_per_step']) for k,v in d['roofline']['per_kernel'].items()})"
done
