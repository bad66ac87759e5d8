#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sgemm_ffma -s 1 -c 1 -o gpurun_out/k3_8192 python tools/prof_configs.py f32 > gpurun_out/k3_8192.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/k3_8192.ncu-rep --page source --csv --print-source sass > gpurun_out/k3_src.csv 2>/dev/null
ncu -i gpurun_out/k3_8192.ncu-rep --page raw --csv > gpurun_out/k3_raw.csv 2>/dev/null
