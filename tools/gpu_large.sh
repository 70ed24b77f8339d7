#!/bin/bash
# long-series path: parity tests, cfg5/cfg3 timings, batch-size sweep, ncu of the four-step kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -x -q > gpurun_out/pytest_long.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_long.log
timeout 600 python tools/bench_micro.py cfg5 cfg3 > gpurun_out/micro.log 2>&1
for per in 16 32 64; do echo "per=$per" >> gpurun_out/micro_per.log; SSA_HANK_PER=$per timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/micro_per.log 2>&1; done
timeout 300 python tools/micro_once.py cfg5 > gpurun_out/micro_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_" -c 3 \
  -o gpurun_out/prof_large python tools/micro_once.py cfg5 > gpurun_out/ncu_large.log 2>&1
echo done
