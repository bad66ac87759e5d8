#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/experiments/ab_bench.py "$@" > gpurun_out/ab.log 2>&1; echo "rc=$?" >> gpurun_out/ab.log
cat gpurun_out/ab.log
