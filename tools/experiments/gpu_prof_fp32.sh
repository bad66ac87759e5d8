#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sgemm_ffma|k_sgemm_3xtf32" -s 1 -c 2 -o gpurun_out/prof_fp32 python tools/experiments/prof_fp32.py 8192 > gpurun_out/ncu_fp32.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_fp32.log
