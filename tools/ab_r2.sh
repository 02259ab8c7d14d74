mkdir -p gpurun_out
for cfg in "PMSZ_PREP2=0" "PMSZ_PREP2=1" "PMSZ_PREP2=1 PMSZ_K0_RULES=1" "PMSZ_PREP2=1 PMSZ_Q_RULES=1"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print(round(d['ms_per_step'],3), {k:(round(v['ms_total_per_step'],3), v['launches_per_step']) for k,v in d['roofline']['per_kernel'].items()})"
done
PMSZ_TAIL_TRACE=1 timeout 300 python tools/one_run.py 512 1 2>&1 | grep -A1 tail1
