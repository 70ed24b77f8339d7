#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/bench_micro.py cfg4 cfg5 > gpurun_out/micro.log 2>&1
SSA_HANK_PER=4 timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/micro.log 2>&1
SSA_HANK_PER=16 timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/micro.log 2>&1
SSA_HANK_PER=32 timeout 300 python tools/bench_micro.py cfg5 >> gpurun_out/micro.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_long.py -x -q -k "matvec or hankel or spectrum" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/bench_micro.py cfg5 > gpurun_out/cfg5_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv \
   python tools/bench_micro.py cfg5 > gpurun_out/ncu_cfg5.log 2>&1
