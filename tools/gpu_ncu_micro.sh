#!/bin/bash
# ncu --set full of the cfg4 matvec kernel and the cfg5 four-step hankelization kernels
mkdir -p gpurun_out
timeout 600 python tools/bench_micro.py cfg4 cfg5 > gpurun_out/micro.log 2>&1
timeout 300 python tools/micro_once.py > gpurun_out/micro_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"matvec|large_" -c 5 \
  -o gpurun_out/prof_micro python tools/micro_once.py > gpurun_out/ncu_micro.log 2>&1
echo done
