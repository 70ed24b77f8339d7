#!/bin/bash
# ncu --set full of the decompose kernels at the bench batch (4096 cfg2 series).
mkdir -p gpurun_out
B=${1:-4096}
timeout 300 python tools/ncu_one.py $B > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|bidiag|hankelize|spectrum" -c 5 \
  -o gpurun_out/prof_cfg2 python tools/ncu_one.py $B > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
