# K0 A/B on the 512^3 bench: 3 runs of the bench line (prep ms per step, total ms per step)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_ab.log 2>&1; echo tests_rc=$?; tail -1 gpurun_out/gputests_ab.log
for i in 1 2 3; do
  python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['roofline']['per_kernel']; print(round(d['ms_per_step'],3), 'prep', round(k['prep']['ms_total_per_step'],3), d['result']['edit_count'])"
done
