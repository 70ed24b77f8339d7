#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hmatrix.py tests/test_gpu_bootstrap.py -q > gpurun_out/pytest_new.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_new.log
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench, paper_0911_4498_b200 as P
print(json.dumps(bench.micro_bootstrap(P)))
print(json.dumps(bench.micro_hmatrix(P)))
" > gpurun_out/new_micro.log 2>&1
echo done
