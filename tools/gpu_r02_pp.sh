#!/bin/bash
# Ping-pong K1 (two consumer groups of 64x128 tiles per CTA): parity, then
# same-process A/B of explicit plans against 128x128 on the shapes VERDICT names.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/pp_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -3 gpurun_out/pp_parity.log; [ $rc -ne 0 ] && exit 1
timeout 1500 python tools/experiments/cfg_ab.py "${SHAPES:-65536,512,512;16384,1024,1024;65536,1024,512;4096,4096,4096;8192,8192,8192;2048,2048,2048;1024,1024,1024;16384,16384,16384}" "128,128,6;64,128,4;128,64,4" 3 > gpurun_out/pp_cfg_ab.jsonl 2> gpurun_out/pp_cfg_ab.err; echo "ab rc=$?"; cat gpurun_out/pp_cfg_ab.jsonl; tail -3 gpurun_out/pp_cfg_ab.err
# mid N: 64x64 with one CTA per SM under stream-K (grid 148) against the chooser's 2-per-SM grid
timeout 900 python tools/experiments/cfg_ab.py "1024,1024,1024;1536,1536,1536;2048,2048,2048;768,768,768" "64,64,4;64,64,4,148;64,128,4;64,128,4,148;128,64,4;128,64,4,148;128,128,6" 3 > gpurun_out/pp_midn.jsonl 2> gpurun_out/pp_midn.err; echo "midn rc=$?"; cat gpurun_out/pp_midn.jsonl; tail -3 gpurun_out/pp_midn.err
