#!/bin/bash
mkdir -p gpurun_out
for ns in 4 8 12 16; do echo "slices=$ns" >> gpurun_out/e2e.log
  SSA_HOST_SLICES=$ns timeout 600 python bench.py --steps 3 --warmup 3 --no-micro --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])" >> gpurun_out/e2e.log 2>&1
done
echo done
