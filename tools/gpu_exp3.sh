#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for e in ${EXPS:-0 1}; do
SSA_LG_EXP=$e SSA_TRACE=1 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3_trace_$e.log 2>&1; echo "exp=$e rc=$?"; tail -22 gpurun_out/cfg3_trace_$e.log | head -8
SSA_LG_EXP=$e timeout 600 python tools/cfg3_bench.py 2>&1 | grep ms=
done
