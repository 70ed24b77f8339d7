#!/bin/bash
mkdir -p gpurun_out
for cfg in "40 8" "56 8" "56 12" "64 12" "56 16"; do set -- $cfg
  echo "first=$1 cap=$2" >> gpurun_out/chk.log
  SSA_FIRST_CHECK=$1 SSA_CHECK_CAP=$2 timeout 300 python tools/prof_cfg2.py 4096 1 4 >> gpurun_out/chk.log 2>&1
done
echo done
