# Round profile set (1 GPU): bench lines, launch list, ncu --set full of K0 and the full sweep.
# usage: bash tools/profile_round.sh TAG
T=${1:-v35}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$T.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests_$T.log
tail -2 gpurun_out/gputests_$T.log
python bench.py > gpurun_out/bench_${T}_default.json 2> gpurun_out/bench_${T}.err; echo default rc=$?
python bench.py --workload hedm > gpurun_out/bench_${T}_hedm.json 2>> gpurun_out/bench_${T}.err; echo hedm rc=$?
python bench.py --impl reference > gpurun_out/bench_${T}_reference.json 2>> gpurun_out/bench_${T}.err; echo reference rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k 'regex:k_prep_q|k_qsweep_tma' -c 2 -o gpurun_out/full_$T \
    python tools/one_run.py 512 1 > gpurun_out/ncu_full_$T.log 2>&1; echo full rc=$?
