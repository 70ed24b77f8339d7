#!/bin/bash
# cfg5 hankelization batch-size sweep (SSA_HANK_PER: terms per batch on each of two streams)
mkdir -p gpurun_out
for per in 8 12 16 24 32 64; do echo "per=$per" >> gpurun_out/per.log; SSA_HANK_PER=$per timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/per.log 2>&1; done
echo done
