# Round-2 final 1-GPU set: tests, smoke, bench lines, launch list.
T=${1:-r02f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_$T.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/gputests_$T.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$T.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke_$T.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${T}_default.json 2> gpurun_out/bench_$T.err; echo default rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_${T}_reference.json 2>> gpurun_out/bench_$T.err; echo reference rc=$?
timeout 600 python bench.py --workload hedm --no-cpu-baseline > gpurun_out/bench_${T}_hedm.json 2>> gpurun_out/bench_$T.err; echo hedm rc=$?
timeout 600 python bench.py --workload strong --no-cpu-baseline --no-dropin > gpurun_out/bench_${T}_strong.json 2>> gpurun_out/bench_$T.err; echo strong rc=$?
timeout 600 python bench.py --f64-original --no-cpu-baseline --no-dropin > gpurun_out/bench_${T}_f64.json 2>> gpurun_out/bench_$T.err; echo f64 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dropin > gpurun_out/ncu_launch_$T.log 2>&1; echo launches rc=$?
for f in default hedm strong f64; do python -c "
import json; d=json.load(open('gpurun_out/bench_${T}_$f.json')); print('$f', round(d['ms_per_step'],3), '%.3e' % d['value'], 'frac', round(d['roofline']['frac'],3), 'e2e', round(d.get('e2e',{}).get('ms_per_step',0),2), 'dropin', d.get('dropin',{}).get('ms_per_call'), d['result'].get('reference_pin'))"; done
python -c "
import json; d=json.load(open('gpurun_out/bench_${T}_reference.json')); print('reference', d['ms_per_step'], d['value'])"
