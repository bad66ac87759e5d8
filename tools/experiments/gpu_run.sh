#!/bin/bash
# Run an arbitrary command on the GPU box with output captured to gpurun_out/run.log.
mkdir -p gpurun_out
timeout ${RUN_TIMEOUT:-300} "$@" > gpurun_out/run.log 2>&1; echo "rc=$?" >> gpurun_out/run.log
tail -80 gpurun_out/run.log
