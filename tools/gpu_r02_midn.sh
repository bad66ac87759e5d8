#!/bin/bash
# Mid N (N=1024 >= 85%): deep-ring 64x64 / 128x64 configs at one CTA per SM
# (64,64,12 and 128,64,8 were compiled in for this experiment only — K1Traits<64,64,2,4,12>,
# K1Traits<128,64,4,2,8> rows in kK1Configs — and dropped after it: not faster.)
# under stream-K, against the compiled configs; explicit plans, bitwise checked.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python tools/experiments/cfg_ab.py "${SHAPES:-1024,1024,1024;768,768,768;1280,1280,1280;1536,1536,1536;2048,2048,2048;3072,3072,3072;4096,4096,4096;65536,512,512}" "${CFGS:-64,64,4;64,64,12;64,64,12,148;128,64,4;128,64,8;128,64,8,148;128,128,6}" 3 > gpurun_out/midn.jsonl 2> gpurun_out/midn.err; echo "ab rc=$?"; cat gpurun_out/midn.jsonl; tail -3 gpurun_out/midn.err
