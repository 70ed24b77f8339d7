#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_par.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_par.log
timeout 300 python tools/prof_cfg2.py 4096 1 4 > gpurun_out/prof_cfg2.log 2>&1
timeout 300 python tools/prof_cfg2.py 4096 1 4 >> gpurun_out/prof_cfg2.log 2>&1
echo done
