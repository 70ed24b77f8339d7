#!/bin/bash
# ncu --set full of one cfg3 Lanczos half-step's FFT kernels (col_fwd, row_cta, col_inv) and
# the reorthogonalization pair (lg_dots, lg_update), plus the cfg4 multi-vector matvec kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python tools/micro_once.py cfg3mv > gpurun_out/cfg3_once.log 2>&1 || { tail gpurun_out/cfg3_once.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lg_col_fwd|lg_row_cta|lg_col_inv|lg_dots|lg_update" \
  --launch-skip 6 -c 3 -o gpurun_out/prof_cfg3fft python tools/micro_once.py cfg3mv > gpurun_out/ncu_cfg3fft.log 2>&1
echo "ncu cfg3 exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"matvec4096" -c 1 --launch-skip 1 \
