#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_lifted_multiproc_gpu.py tests/test_bench_multirank_gpu.py tests/test_lifted.py -q -x -rf > gpurun_out/r02_direct.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/r02_direct.log
