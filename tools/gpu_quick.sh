#!/bin/bash
# quick GPU pass: build, selected tests ($TESTS), cfg3 timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -q -m gpu -x > gpurun_out/gputest_quick.log 2>&1
  echo "pytest rc=$?"; tail -30 gpurun_out/gputest_quick.log
fi
timeout 600 python tools/cfg3_bench.py > gpurun_out/cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -20 gpurun_out/cfg3.log
if [ -n "$NCU3" ]; then
  timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python tools/cfg3_once.py > gpurun_out/ncu3.log 2>&1
  echo "ncu rc=$?"
fi
