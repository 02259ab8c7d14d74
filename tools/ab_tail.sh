# k_tail grid size A/B (PMSZ_TAIL_BLOCKS) with per-iteration device timestamps
mkdir -p gpurun_out
for nb in 0 32 8 1; do
  echo "== nb $nb"
  PMSZ_TAIL_BLOCKS=$nb PMSZ_TAIL_TRACE=1 python tools/one_run.py 512 2 2>&1 | tail -5
  PMSZ_TAIL_BLOCKS=$nb python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['roofline']['per_kernel']; print('nb $nb', round(d['ms_per_step'],3), 'tail', round(k['tail']['ms_total_per_step'],3), k['tail']['launches_per_step'], d['result']['edit_count'])"
done
