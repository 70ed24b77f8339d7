#!/bin/bash
# Round snapshot: tests, smoke, full bench (with CPU baseline and microbenchmarks),
# reference arm, launch list of one bench step, ncu --set full of the dominant kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?" >> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/ncu_one.py 4096 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|hankelize|spectrum" -c 4 \
  -o gpurun_out/prof_round python tools/ncu_one.py 4096 > gpurun_out/ncu_full.log 2>&1
echo done
