#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/bench_configs.py "$@" > gpurun_out/configs.json 2> gpurun_out/configs.err; echo "rc=$?" >> gpurun_out/configs.err
tail -5 gpurun_out/configs.err
