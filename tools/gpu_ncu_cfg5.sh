#!/bin/bash
# cfg5 Hankelization at HEAD: parity tests of the H = 2^16 / 2^17 path, the bench line,
# ncu --set full of the three kernels of one 64-term batch -> gpurun_out/cfg5/.
O=gpurun_out/cfg5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "long or bounds or hankel" > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -2 $O/pytest.log
timeout 600 python tools/micro_lines.py cfg5 > $O/micro.log 2>&1; echo "micro exit $?"; cut -c1-700 $O/micro.log
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"lg_col16|lg_row_warp" -c 6 \
  -o /tmp/prof_cfg5 python tools/micro_once.py cfg5 > $O/ncu_cfg5.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py /tmp/prof_cfg5.ncu-rep $O/ncu_r02_cfg5_summary.json --batch 1 \
  --note "tools/micro_once.py cfg5: the four-step Hankelization kernels of one 64-term batch at N = 2^18 (lg_col16_fwd: u and v columns, lg_row_warp: row pairs + product, lg_col16_hank: inverse columns + sigma/c epilogue); ncu --set full --clock-control none" > /dev/null 2>&1
python tools/ncu_stalls.py /tmp/prof_cfg5.ncu-rep > $O/ncu_r02_cfg5_stalls.txt 2>&1
ls $O; echo done
