#!/bin/bash
# ncu --set full of the cfg3-size four-step correlation kernels (col_fwd, row_cta, col_inv;
# a plain ssa_matvec at N = 2^20: the Lanczos loop itself is a graph with conditional nodes,
# which ncu cannot profile per kernel) and of the cfg4 multi-vector matvec kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python tools/micro_once.py cfg3mv > gpurun_out/cfg3_once.log 2>&1 || { tail gpurun_out/cfg3_once.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_col_fwd|lg_row_cta|lg_col_inv|lg_dots|lg_update" \
  --launch-skip 6 -c 3 -o gpurun_out/prof_cfg3fft python tools/micro_once.py cfg3mv > gpurun_out/ncu_cfg3fft.log 2>&1
echo "ncu cfg3 exit $?"
timeout 300 python tools/micro_once.py cfg4m > gpurun_out/micro_once.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec4096" -c 1 --launch-skip 1 \
  -o gpurun_out/prof_cfg4m python tools/micro_once.py cfg4m > gpurun_out/ncu_cfg4m.log 2>&1
echo "ncu cfg4m exit $?"
