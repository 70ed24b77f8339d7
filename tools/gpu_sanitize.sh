#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md): run every small workload
# of tools/sanitize_workload.py under that tool, summary lines into gpurun_out/.
#   gpurun --timeout 1800 -- bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck|initcheck [workloads...]
tool=$1; shift
wl=${*:-"cfg1 cfg2b8 cfg4b64 long4096 hank hmatrix bootstrap"}
mkdir -p gpurun_out/san
python -c "import __graft_entry__ as g; g.build()" || exit 1
for w in $wl; do
  # plain run first: the sanitizer only runs on a workload that exited 0 without it
  if ! timeout 300 python tools/sanitize_workload.py $w > gpurun_out/san/${tool}_${w}.plain 2>&1; then
    echo "$w: plain run failed" | tee -a gpurun_out/san/${tool}_summary.txt; continue
  fi
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python tools/sanitize_workload.py $w > gpurun_out/san/${tool}_${w}.log 2>&1
  rc=$?
  echo "$w: rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/${tool}_${w}.log | tr '\n' ' ')" | tee -a gpurun_out/san/${tool}_summary.txt
done
