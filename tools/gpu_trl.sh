#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_trl.py -q -m gpu -x -s ${PYTEST_ARGS} > gpurun_out/gputest_trl.log 2>&1
echo "pytest rc=$?"; grep -E "TRL|passed|failed|Error|assert" gpurun_out/gputest_trl.log | head -40; tail -30 gpurun_out/gputest_trl.log
