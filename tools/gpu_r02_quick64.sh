#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gather.py -q -x > gpurun_out/r02_parity3.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_parity3.log
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "768,768,768;1024,1024,1024;65536,512,512;8192,8192,8192" ab/libmoa_r01.so ab/libmoa_nolag.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_r01b.jsonl 2>&1; echo "ab rc=$?"; cut -c1-200 gpurun_out/r02_ab_r01b.jsonl
