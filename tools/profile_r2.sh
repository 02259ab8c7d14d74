# Round-2 profile set (1 GPU): launch list of one bench step + ncu --set full of every kernel >= 5 % of a step.
T=${1:-r02}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-dropin > gpurun_out/ncu_launch_$T.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on \
    -k 'regex:k_prep_q|k_qsweep_tma|k_apply_list|k_defer|k_tail|k_chunk_list|k_chunk_write|k_chunk_count_scan|k_sweep_list|k_mark_list' \
    -c 34 -o gpurun_out/full_$T python tools/one_run.py 512 1 > gpurun_out/ncu_full_$T.log 2>&1; echo full rc=$?
