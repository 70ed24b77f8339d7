#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_long.py -x -q > gpurun_out/pytest_long.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_long.log
timeout 600 python tools/bench_micro.py cfg3 > gpurun_out/micro.log 2>&1
timeout 300 python tools/cfg3_once.py > gpurun_out/cfg3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python tools/cfg3_once.py > gpurun_out/ncu_cfg3.log 2>&1
echo done
