#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "interleaved or run_host" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_micro.py cfg5 > gpurun_out/cfg5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"large_" -s 4 -c 3 \
  -o gpurun_out/prof_cfg5 python tools/bench_micro.py cfg5 > gpurun_out/ncu_cfg5.log 2>&1
timeout 300 python tools/cfg3_once.py > gpurun_out/cfg3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python tools/cfg3_once.py > gpurun_out/ncu_cfg3.log 2>&1
