#!/bin/bash
# Quick GPU iteration: selected tests (TESTS env) + optional bench args.
mkdir -p gpurun_out
timeout 900 python -m pytest ${TESTS:-tests} -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then timeout 900 python $BENCH > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err; echo "bench rc=$?"; cat gpurun_out/quick_bench.json; tail -5 gpurun_out/quick_bench.err; fi
