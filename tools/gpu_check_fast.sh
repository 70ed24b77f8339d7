#!/bin/bash
# Checkpoint call, fast things first: build, default bench, smoke, ncu --set full of the cfg5
# kernels, then all GPU tests.  Outputs under gpurun_out/check/.
O=gpurun_out/check; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"; tail -c 300 $O/bench.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lg_col16|lg_row_warp" -c 6 \
  -o /tmp/prof_cfg5 python tools/micro_once.py cfg5 > $O/ncu_cfg5.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py /tmp/prof_cfg5.ncu-rep $O/ncu_r02_cfg5_summary.json --batch 1 \
  --note "tools/micro_once.py cfg5: the four-step Hankelization kernels of one 16-term batch at N = 2^18 (lg_col16_fwd: u and v columns, 8 columns per CTA; lg_row_warp: row pairs + product; lg_col16_hank: inverse columns + sigma/c epilogue); ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_cfg5.ncu-rep > $O/ncu_r02_cfg5_stalls.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
