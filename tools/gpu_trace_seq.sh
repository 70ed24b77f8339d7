#!/bin/bash
# cfg3 kernel timeline: per-id totals and a window of the raw start sequence (SSA_TRACE_SEQ)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
SSA_TRACE=1 SSA_TRACE_SEQ=${SEQ:-2000} timeout 300 python tools/cfg3_once.py ${REORTH:-1} > gpurun_out/cfg3_seq.log 2>&1; echo "rc=$?"
cat gpurun_out/cfg3_seq.log | cut -c1-200 | tail -70
