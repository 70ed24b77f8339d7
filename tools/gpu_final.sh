#!/bin/bash
# (ncu reports stay in /tmp on the box: only their summaries travel back, gpurun_out <= 64 MiB)
# Round snapshot: all GPU tests, smoke, full bench (micro lines, CPU baseline), reference arm,
# launch list of one bench step, ncu --set full of the dominant kernel and the micro kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?" >> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/ncu_one.py 4096 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|hankelize|spectrum" -c 4 \
  -o /tmp/prof_round python tools/ncu_one.py 4096 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_round.ncu-rep gpurun_out/ncu_cfg2_summary.json --batch 4096 \
  --note "one cfg2 decompose+reconstruct of 4096 series (tools/ncu_one.py), ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_round.ncu-rep > gpurun_out/ncu_cfg2_stalls.txt 2>&1
timeout 300 python tools/micro_once.py > gpurun_out/micro_once.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_|matvec4096" -c 4 \
  -o /tmp/prof_micro python tools/micro_once.py > gpurun_out/ncu_micro.log 2>&1
python tools/ncu_summary.py /tmp/prof_micro.ncu-rep gpurun_out/ncu_micro_summary.json --batch 1 \
  --note "tools/micro_once.py: cfg4 matvec4096_kernel (4096 series, one X v) and cfg5 four-step kernels (64-term batch); ncu --set full --clock-control none (caches flushed between kernels)" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_micro.ncu-rep > gpurun_out/ncu_micro_stalls.txt 2>&1
timeout 300 python tools/cfg3_once.py > gpurun_out/cfg3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python tools/cfg3_once.py > gpurun_out/ncu_cfg3.log 2>&1
echo done
