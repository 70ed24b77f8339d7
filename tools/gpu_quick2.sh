#!/bin/bash
# selected GPU tests ($TESTS) + bench line without extras
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest ${TESTS:-tests/test_gpu_parity.py} -q -m gpu -x > gpurun_out/gputest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_q.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-micro --no-fro --no-overshoot --no-trl > gpurun_out/bench_q.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print('value', d['value'], 'ms', d['ms_per_step'], 'phase', d['phase_ms'], 'ritz', d['ritz_roofline']['frac'], 'cfg3', d.get('decompose_cfg3',{}).get('ms'))"
