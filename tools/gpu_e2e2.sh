#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "run_host" > gpurun_out/pytest_rh.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_rh.log
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-micro --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" >> gpurun_out/e2e.log 2>&1; done
echo done
