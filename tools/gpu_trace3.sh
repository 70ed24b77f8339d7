#!/bin/bash
# cfg3 time breakdown by traced kernel (SSA_TRACE) + graph / grid-sync overheads
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 120 ./tools/graph_overhead 2>&1 | tee gpurun_out/graph_overhead.txt
SSA_TRACE=1 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3_trace.log 2>&1; echo "rc=$?"; tail -60 gpurun_out/cfg3_trace.log
