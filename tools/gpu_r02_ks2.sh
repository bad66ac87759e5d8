#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/r02_parity_ks2.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -1 gpurun_out/r02_parity_ks2.log; [ $rc -ne 0 ] && exit 1
timeout 900 python tools/experiments/cfg_ab.py "768,768,768;1024,1024,1024;1536,1536,1536;2048,2048,2048;4096,4096,4096;65536,512,512;16384,1024,1024" "64,64,4;64,64,6;128,64,4;128,64,6;64,32,4;128,128,6" 3 | tee gpurun_out/r02_cfg_ab_ks2.jsonl
SHAPES="8192,8192,8192;65536,512,512;16384,1024,1024;4096,4096,4096;2048,2048,2048" LIBS="paper_2306_11148_b200/libmoa.so ab/libmoa_ks128.so" OUT=r02_ab_ks128 bash tools/gpu_r02_ab.sh
