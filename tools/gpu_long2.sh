#!/bin/bash
# long path: its tests, then the cfg3 trace and timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
SSA_TRACE=1 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3_trace.log 2>&1; echo "trace rc=$?"; tail -24 gpurun_out/cfg3_trace.log
timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3.log 2>&1; echo "cfg3 rc=$?"; cat gpurun_out/cfg3.log
timeout 1500 python -m pytest tests/test_gpu_long.py tests/test_gpu_edge.py -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/gputest_long.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/gputest_long.log
