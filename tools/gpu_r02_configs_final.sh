#!/bin/bash
# Every BASELINE config with the final code (tools/bench_configs.py, all sections).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python tools/bench_configs.py > gpurun_out/cfgfinal.json 2> gpurun_out/cfgfinal.err; echo "configs rc=$?"; tail -3 gpurun_out/cfgfinal.err
