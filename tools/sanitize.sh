#!/bin/sh
# compute-sanitizer over every kernel family (tools/sanitize_driver.py); logs in gpurun_out/
# racecheck runs without the captured-graph replay (SKIP_GRAPH=1): racecheck
# crashes the process on a graph with a conditional node (memcheck, synccheck
# and initcheck run it); the kernels inside the branches are the radix passes
# the rest of the driver runs directly.
CS=compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  skip=""; [ $tool = racecheck ] && skip=1
  SKIP_GRAPH=$skip timeout 1500 $CS --tool $tool --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tail -1)"
done
timeout 1500 $CS --tool memcheck --print-limit 20 python tools/sanitize_driver.py waves > gpurun_out/sanitize_memcheck_waves.log 2>&1
echo "memcheck waves rc=$? $(grep 'ERROR SUMMARY' gpurun_out/sanitize_memcheck_waves.log | tail -1)"
