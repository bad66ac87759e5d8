#!/bin/bash
# 128x128 ring depth 3/4/5/6 (experiment; could a smaller ring free shared memory for a
# (the 3/4/5-stage 128x128 configs were compiled in for this experiment only and dropped)
# staged tile epilogue?). Explicit plans, bitwise checked.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python tools/experiments/cfg_ab.py "65536,512,512;16384,1024,1024;8192,8192,8192;4096,4096,4096;16384,16384,16384" "128,128,6;128,128,5;128,128,4;128,128,3" 3 > gpurun_out/stages_ab.jsonl 2> gpurun_out/stages_ab.err; echo "ab rc=$?"; cat gpurun_out/stages_ab.jsonl; tail -3 gpurun_out/stages_ab.err
