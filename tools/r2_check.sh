# Round-2 GPU check: tests, smoke, default bench (1 GPU).  usage: bash tools/r2_check.sh TAG [pytest-args]
T=${1:-r2}
shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/gputests_$T.log 2>&1; echo tests_rc=$? >> gpurun_out/gputests_$T.log
tail -3 gpurun_out/gputests_$T.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$T.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err; echo bench rc=$?
tail -c 600 gpurun_out/bench_${T}.json
