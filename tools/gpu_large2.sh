#!/bin/bash
mkdir -p gpurun_out
for per in 16 32 64 128; do echo "per=$per" >> gpurun_out/micro_per.log; SSA_HANK_PER=$per timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/micro_per.log 2>&1; done
echo done
