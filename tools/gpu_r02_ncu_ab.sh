#!/bin/bash
# ncu --set full of K1 at 8192^3 with the round-1 build and the current build (stall reasons)
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in r01; do
  lib=paper_2306_11148_b200/libmoa.so; [ $v = r01 ] && lib=ab/libmoa_r01.so
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dgemm_tma -s 1 -c 1 -o gpurun_out/ab8k_$v python tools/experiments/one_gemm.py $lib 8192 8192 8192 > gpurun_out/ab8k_$v.log 2>&1; echo "$v rc=$?"
  ncu -i gpurun_out/ab8k_$v.ncu-rep --page raw --csv > gpurun_out/ab8k_$v.raw.csv 2>/dev/null
done
