#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_dgemm_tma -s 2 -c 4 -o gpurun_out/prof_small python tools/prof_small.py ${1:-2048} > gpurun_out/ncu_small.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_small.log
