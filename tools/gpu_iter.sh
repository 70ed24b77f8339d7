#!/bin/bash
# one iteration: smoke, gpu tests, cfg2 profile, micro (cfg4/cfg5), ncu of lanczos
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python tools/prof_cfg2.py 4096 1 4 > gpurun_out/prof_cfg2.log 2>&1
timeout 600 python tools/bench_micro.py cfg4 cfg5 > gpurun_out/micro.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
if [ "$1" == "ncu" ]; then
timeout 300 python tools/ncu_one.py 4096 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lanczos" -c 1 \
  -o gpurun_out/prof_iter python tools/ncu_one.py 4096 > gpurun_out/ncu_full.log 2>&1
fi
