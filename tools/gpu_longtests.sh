#!/bin/bash
# long-path + edge GPU tests only
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_long.py tests/test_gpu_edge.py -q -m gpu -x ${PYTEST_ARGS} > gpurun_out/gputest_long.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/gputest_long.log
