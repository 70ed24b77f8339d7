#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "matvec or spectrum" > gpurun_out/pytest_mv.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_mv.log
timeout 600 python tools/bench_micro.py cfg4 > gpurun_out/micro.log 2>&1
SSA_MATVEC_SMEM=1 timeout 600 python tools/bench_micro.py cfg4 >> gpurun_out/micro.log 2>&1
timeout 300 python tools/micro_once.py cfg4 > gpurun_out/micro_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"matvec" -c 2 \
  -o gpurun_out/prof_mv python tools/micro_once.py cfg4 > gpurun_out/ncu_mv.log 2>&1
echo done
