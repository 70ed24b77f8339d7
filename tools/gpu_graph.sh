#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
./tools/graph_overhead 2>&1 | tee gpurun_out/graph_overhead.txt
SSA_DEBUG=1 timeout 600 python tools/cfg3_bench.py 2>&1 | tee gpurun_out/cfg3.log
SSA_DEBUG=1 SSA_LG_NOPDL=1 timeout 600 python tools/cfg3_bench.py 2>&1 | tee gpurun_out/cfg3_nopdl.log
