#!/bin/bash
# tests of the long path, full bench (with micro lines and CPU baseline), ncu of cfg5/cfg4 kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -x -q > gpurun_out/pytest_long.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_long.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?" >> gpurun_out/bench_full.err
timeout 300 python tools/micro_once.py > gpurun_out/micro_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_|matvec4096" -c 4 \
  -o gpurun_out/prof_micro python tools/micro_once.py > gpurun_out/ncu_micro.log 2>&1
echo done
