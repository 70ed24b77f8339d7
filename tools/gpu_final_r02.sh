#!/bin/bash
# Round-2 checkpoint at HEAD: all GPU tests, smoke, full bench + reference arm, cfg2 launch
# list, ncu --set full summaries (cfg2 step kernels; cfg4 multi-vector matvec, cfg5 and cfg3
# four-step kernels, cfg3 Ritz), cfg3 SSA_TRACE timeline.  Outputs under gpurun_out/final/.
O=gpurun_out/final; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?"; tail -c 300 $O/bench.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
   python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-micro --no-fro --no-trl --no-overshoot > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_cfg2.csv $O/launches_cfg2.json > $O/launches_cfg2.txt 2>&1
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lanczos|ritz|hankelize|spectrum" -c 4 \
  -o /tmp/prof_cfg2 python tools/ncu_one.py 4096 3 > $O/ncu_cfg2.log 2>&1
python tools/ncu_summary.py /tmp/prof_cfg2.ncu-rep $O/ncu_r02_cfg2_summary.json --batch 4096 \
  --note "one cfg2 decompose+reconstruct of 4096 series (tools/ncu_one.py, PRO default), ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_cfg2.ncu-rep > $O/ncu_r02_cfg2_stalls.txt 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lg_col|lg_row|matvec4096" -c 12 \
  -o /tmp/prof_micro python tools/micro_once.py cfg4m cfg5 cfg3mv > $O/ncu_micro.log 2>&1
python tools/ncu_summary.py /tmp/prof_micro.ncu-rep $O/ncu_r02_micro_summary.json --batch 1 \
  --note "tools/micro_once.py cfg4m cfg5 cfg3mv: matvec4096_kernel (ssa_matvec_multi, 2048 series x 32 vectors), cfg5 four-step kernels (64-term batch), cfg3-size four-step correlation (one item); ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_micro.ncu-rep > $O/ncu_r02_micro_stalls.txt 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lg_col16|lg_row_warp" -c 6 \
  -o /tmp/prof_cfg5 python tools/micro_once.py cfg5 > $O/ncu_cfg5.log 2>&1
python tools/ncu_summary.py /tmp/prof_cfg5.ncu-rep $O/ncu_r02_cfg5_summary.json --batch 1 \
  --note "tools/micro_once.py cfg5: the four-step Hankelization kernels of one 64-term batch at N = 2^18 (lg_col16_fwd: u and v columns, lg_row_warp: row pairs + product, lg_col16_hank: inverse columns + sigma/c epilogue); ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_cfg5.ncu-rep > $O/ncu_r02_cfg5_stalls.txt 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"lg_ritz" -c 2 -o /tmp/prof_lgritz python tools/cfg3_once.py > $O/ncu_lgritz.log 2>&1
python tools/ncu_stalls.py /tmp/prof_lgritz.ncu-rep > $O/ncu_r02_lgritz_stalls.txt 2>&1
SSA_TRACE=1 timeout 300 python tools/cfg3_once.py > $O/cfg3_trace.log 2>&1
ls $O; echo done
