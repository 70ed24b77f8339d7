#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "decompose" > gpurun_out/pytest_ritz.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ritz.log
for i in 1 2; do timeout 300 python tools/prof_cfg2.py 4096 1 4 2>&1 | grep decompose >> gpurun_out/ritz.log; done
echo done
