#!/bin/bash
# ncu --set full: lanczos/ritz/hankelize at the bench batch (4096 cfg2 series) and the
# cfg4-shaped matvec kernel (4096 series).
mkdir -p gpurun_out
timeout 300 python tools/ncu_one.py 4096 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|hankelize|spectrum|bidiag" -c 5 \
  -o gpurun_out/prof_cfg2_v4 python tools/ncu_one.py 4096 > gpurun_out/ncu_full.log 2>&1
echo "ncu1 exit $?" >> gpurun_out/ncu_full.log
timeout 300 python tools/ncu_matvec.py 4096 > gpurun_out/ncu_plain2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec" -c 1 \
  -o gpurun_out/prof_matvec python tools/ncu_matvec.py 4096 > gpurun_out/ncu_full2.log 2>&1
echo "ncu2 exit $?" >> gpurun_out/ncu_full2.log
