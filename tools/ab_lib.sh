# A/B of the default build against paper_2601_01787_b200/_lib/ab/libpmsz.so (PMSZ_LIB) on the 512^3 bench
mkdir -p gpurun_out
one() {
  python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['roofline']['per_kernel']; print('$1', round(d['ms_per_step'],3), 'prep', round(k['prep']['ms_total_per_step'],3), d['result']['edit_count'])"
}
for i in 1 2; do one base; PMSZ_LIB=$PWD/paper_2601_01787_b200/_lib/ab/libpmsz.so one alt; done
