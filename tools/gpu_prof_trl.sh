#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/prof_trl.py 1024 40 20 2>&1 | tee gpurun_out/prof_trl.log
timeout 600 python tools/prof_cfg2.py 1024 1 2>&1 | tail -12 | tee gpurun_out/prof_fro.log
