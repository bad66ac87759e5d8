#!/bin/bash
mkdir -p gpurun_out/sanitizer
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/r02_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitizer/r02_$t.log
done
