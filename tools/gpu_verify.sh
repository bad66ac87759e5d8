#!/bin/bash
# tests + A/B vs a saved older build + config sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
if [ -n "$1" ]; then timeout 900 python tools/experiments/ab_bench.py "$1" paper_2306_11148_b200/libmoa.so > gpurun_out/ab.log 2>&1; cat gpurun_out/ab.log; fi
timeout 1200 python tools/bench_configs.py --sizes 1024,1536,2048,3072,4096,6144,8192,16384 > gpurun_out/configs.json 2> gpurun_out/configs.err; echo "configs rc=$?"
