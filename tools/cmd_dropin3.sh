#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_di.log 2>&1 || { tail -20 gpurun_out/build_di.log; exit 1; }
timeout 900 python -m pytest tests/test_integration_stub.py tests/test_gpu_parity.py tests/test_parallel_api.py -x -q -m gpu > gpurun_out/gputests_di.log 2>&1
echo tests=$?; tail -3 gpurun_out/gputests_di.log
timeout 600 python tools/dropin_parallel.py 2>&1 | grep -v Warn | tee gpurun_out/dropin_parallel.log
