#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python tools/prof_cfg2.py 4096 1 4 > gpurun_out/prof_cfg2.log 2>&1
timeout 600 python tools/bench_micro.py cfg4 cfg5 cfg3 > gpurun_out/micro.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/ncu_matvec.py 4096 > gpurun_out/ncu_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec" -c 1 \
  -o gpurun_out/prof_matvec_v6 python tools/ncu_matvec.py 4096 > gpurun_out/ncu_full2.log 2>&1
