#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -x -q -k "hankelize or cfg5" > gpurun_out/pytest_long.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_long.log
for i in 1 2; do timeout 600 python tools/bench_micro.py cfg5 >> gpurun_out/micro.log 2>&1; done
echo done
