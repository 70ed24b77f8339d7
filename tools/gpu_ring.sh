#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_cfg1.py > gpurun_out/p1.log 2>&1
timeout 600 python -c "
import sys, json; sys.path.insert(0, '.')
import bench, paper_0911_4498_b200 as P
print(json.dumps(bench.micro_decompose_cfg1(P)))
print(json.dumps(bench.micro_bootstrap(P)))
print(json.dumps(bench.micro_hmatrix(P)))
" > gpurun_out/new_micro.log 2>&1
timeout 600 python tools/prof_cfg2.py 4096 1 4 > gpurun_out/prof_cfg2.log 2>&1
echo done
