#!/bin/bash
# thick restart: parity tests + bench trl line only
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_trl.py -q -m gpu -x > gpurun_out/gputest_trl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_trl.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-micro --no-fro --no-overshoot > gpurun_out/bench_trl.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_trl.log').read().strip().splitlines()[-1]); print('PRO', d['value'], 'TRL', json.dumps(d['trl']))"
