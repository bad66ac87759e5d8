#!/bin/bash
# 80x96 tiles (143 tiles at N = 1024: one wave on 143 of 148 SMs): parity of every
# K1 config, then explicit-plan A/B against the chooser's tiles around N = 1024 and at
# large N (its eta).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x -k "each_compiled or stream_k or latency" > gpurun_out/t8096_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -2 gpurun_out/t8096_parity.log; [ $rc -ne 0 ] && exit 1
timeout 1500 python tools/experiments/cfg_ab.py "1024,1024,1024;960,960,960;1040,1040,1040;1152,1152,1152;1280,1280,1280;2048,2048,2048;4096,4096,4096;16384,16384,16384;1024,4096,1024;65536,512,512" "80,96,8;128,64,4;64,64,4;128,128,6" 3 > gpurun_out/t8096_ab.jsonl 2> gpurun_out/t8096_ab.err; echo "ab rc=$?"; cat gpurun_out/t8096_ab.jsonl; tail -3 gpurun_out/t8096_ab.err
