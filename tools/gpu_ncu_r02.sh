#!/bin/bash
# Round-2 profiles at HEAD: fp64 peaks (burst + sustained, with clocks), cfg2 launch list,
# ncu --set full of the cfg2 step kernels and of the cfg4 / cfg5 kernels, cfg3 (graph: only
# the kernels outside the loop are visible to ncu; SSA_TRACE timeline instead)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 250 > gpurun_out/peaks_clocks.csv 2>&1 &
SMI=$!
./tools/peaks > gpurun_out/peaks.json 2> gpurun_out/peaks.err; sleep 1; kill $SMI 2>/dev/null
cat gpurun_out/peaks.json
timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-fro --no-trl --no-overshoot > gpurun_out/plain.log 2>&1 && \
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-fro --no-trl --no-overshoot > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_cfg2.csv gpurun_out/launches_cfg2.json | head -12
timeout 300 python tools/ncu_one.py 4096 3 > gpurun_out/ncu_plain.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|hankelize|spectrum" -c 4 \
  -o /tmp/prof_round python tools/ncu_one.py 4096 3 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/prof_round.ncu-rep gpurun_out/ncu_r02_cfg2_summary.json --batch 4096 \
  --note "one cfg2 decompose+reconstruct of 4096 series (tools/ncu_one.py, PRO default), ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_round.ncu-rep > gpurun_out/ncu_r02_cfg2_stalls.txt 2>&1
timeout 300 python tools/micro_once.py > gpurun_out/micro_once.log 2>&1 && \
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lg_|matvec4096" -c 4 \
  -o /tmp/prof_micro python tools/micro_once.py > gpurun_out/ncu_micro.log 2>&1
python tools/ncu_summary.py /tmp/prof_micro.ncu-rep gpurun_out/ncu_r02_micro_summary.json --batch 1 \
  --note "tools/micro_once.py: cfg4 matvec4096_kernel (4096 series, one X v) and cfg5 four-step kernels (64-term batch); ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_micro.ncu-rep > gpurun_out/ncu_r02_micro_stalls.txt 2>&1
SSA_TRACE=1 timeout 300 python tools/cfg3_once.py > gpurun_out/cfg3_trace.log 2>&1
ls -la gpurun_out
echo done
