#!/bin/bash
mkdir -p gpurun_out
timeout 300 python "$@" > gpurun_out/dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dbg.log
cat gpurun_out/dbg.log | tail -60
