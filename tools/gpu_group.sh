#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "grouped or hankelize or reconstruct" > gpurun_out/pytest_grp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_grp.log
timeout 900 python -m pytest tests/test_gpu_long.py -q -k "h8192" > gpurun_out/pytest_h8192.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_h8192.log
echo done
