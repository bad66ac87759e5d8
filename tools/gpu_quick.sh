#!/bin/bash
# Quick GPU iteration: tests given as arguments (default: all gpu tests).
mkdir -p gpurun_out
timeout 900 python -m pytest "${@:-tests}" -x -q -m gpu -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -40 gpurun_out/pytest_gpu.log
