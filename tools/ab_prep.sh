# A/B of the z-chunk of K0 (PMSZ_PREP_ZCHUNK) on the 512^3 and HEDM benches
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests4.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests4.log
tail -2 gpurun_out/gputests4.log
one() {
  python bench.py --no-e2e --no-cpu-baseline $2 > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['roofline']['per_kernel']; print('$1', round(d['ms_per_step'],3), 'prep', round(k['prep']['ms_total_per_step'],3), d['result'].get('edit_count'))"
}
one default ""
PMSZ_PREP_ZCHUNK=64 one hedm64 "--workload hedm"
one hedm_default "--workload hedm"
PMSZ_PREP_ZCHUNK=16 one hedm16 "--workload hedm"
