#!/bin/bash
# Experiment call: build, selected GPU tests ($TESTS), cfg5 A/B of an env knob ($AB: parity
# tests with it set, then tools/cfg5_ab.py), cfg5 sweep ($PERS), micro lines ($LINES).
O=gpurun_out/exp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > $O/pytest.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest.log
fi
if [ -n "$AB" ]; then
  env $AB=1 timeout 900 python -m pytest tests -m gpu -q -x -k "cfg5_shape or radix16 or many_batches" > $O/pytest_ab.log 2>&1; echo "pytest ($AB=1) exit $?"; tail -2 $O/pytest_ab.log
  timeout 600 python tools/cfg5_ab.py $AB ${ABR:-3} > $O/ab.txt 2>&1; echo "ab exit $?"; tail -8 $O/ab.txt
fi
if [ -n "$PERS" ]; then timeout 600 python tools/cfg5_sweep.py $PERS > $O/sweep.txt 2>&1; echo "sweep exit $?"; cat $O/sweep.txt | tail -8; fi
if [ -n "$LINES" ]; then timeout 900 python tools/micro_lines.py $LINES > $O/micro.log 2>&1; echo "micro exit $?"; cut -c1-900 $O/micro.log; fi
if [ -n "$NCU" ]; then
  timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none -k regex:"$NCU" -c ${NCUC:-3} python tools/micro_once.py ${NCUW:-cfg5} > $O/ncu.txt 2>&1; echo "ncu exit $?"; grep -E "lg_|matvec|duration|fp64|warps|registers|dfma|dadd|dmul" $O/ncu.txt | head -40
fi
