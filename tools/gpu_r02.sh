#!/bin/bash
# round-2 GPU pass: build, the GPU tests, one bench line (default arguments)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -q -m gpu ${PYTEST_ARGS} > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -30 gpurun_out/gputest.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 6000 gpurun_out/bench.log; tail -20 gpurun_out/bench.err
