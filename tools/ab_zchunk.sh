for zc in 16 20 24 32; do
  PMSZ_PREP_ZCHUNK=$zc python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['roofline']['per_kernel']; print('zc $zc', round(d['ms_per_step'],3), 'prep', round(k['prep']['ms_total_per_step'],3))"
done
