#!/bin/bash
# cfg3 diagnosis: PRO/FRO timings with and without PDL, then the ncu launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
SSA_DEBUG=1 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3.log 2>&1; echo "cfg3 rc=$?"; cat gpurun_out/cfg3.log
SSA_DEBUG=1 SSA_LG_NOPDL=1 timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3_nopdl.log 2>&1; echo "nopdl rc=$?"; cat gpurun_out/cfg3_nopdl.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/cfg3_once.py > gpurun_out/ncu3.log 2>&1
echo "ncu rc=$?"; python tools/launch_summary.py gpurun_out/launches_cfg3.csv gpurun_out/launches_cfg3.json | head -40
