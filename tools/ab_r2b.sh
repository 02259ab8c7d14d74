mkdir -p gpurun_out
for cfg in "PMSZ_PREP2=0" "PMSZ_PREP2=1" "PMSZ_PREP2=1 PMSZ_LIB=tools/ablib/libpmsz_minb3.so"; do
  echo "== $cfg"
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/ab.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print(round(d['ms_per_step'],3), {k:(round(v['ms_total_per_step'],3), v['launches_per_step']) for k,v in d['roofline']['per_kernel'].items()})"
done
PMSZ_PREP2=1 ncu --set full --clock-control none --import-source on -k regex:k_prep2 -c 1 -o gpurun_out/prep2_r2 python tools/one_run.py 512 1 > gpurun_out/ncu_prep2.log 2>&1; echo ncu=$?
