#!/bin/bash
# Runs the fp64 probe on the GPU box with clocks sampled alongside.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/probe_nvidia_smi.txt 2>&1
nproc > gpurun_out/probe_host.txt; lscpu | grep "Model name" >> gpurun_out/probe_host.txt
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 200 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/fp64_probe | tee gpurun_out/probe_fp64.jsonl
kill $SMI
