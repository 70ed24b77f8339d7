#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
SSA_TRACE=1 SSA_TRACE_SEQ=1200 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3_seq.log 2>&1; echo "rc=$?"; grep "ssa seq" gpurun_out/cfg3_seq.log | head -40
