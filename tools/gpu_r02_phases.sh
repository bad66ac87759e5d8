#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for pl in "16,16,4" "16,16,8" "16,32,4" "16,32,8"; do
  PHASES_PLAN=$pl timeout 300 python tools/experiments/phases.py ab/libmoa_phases.so 128,256,512 2>&1 | sed "s/^/$pl /"
done | tee gpurun_out/r02_phases_ks.txt
