#!/bin/bash
# Iteration call: build, selected GPU tests ($TESTS, pytest -k expression), micro lines ($LINES).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > gpurun_out/pytest_iter.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/pytest_iter.log
fi
if [ -n "$LINES" ]; then
  timeout 900 python tools/micro_lines.py $LINES > gpurun_out/micro_iter.log 2>&1; echo "micro exit $?"; cut -c1-1500 gpurun_out/micro_iter.log
fi
