mkdir -p gpurun_out; timeout 900 python -m pytest tests/test_integration_stub.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gputests_r2n.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_r2n.log
PMSZ_E2E_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-dropin --steps 5 2>&1 | grep -E "e2e:" | tail -3
