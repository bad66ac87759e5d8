#!/bin/bash
# Per-rank compute of configs[4] at G = 1/2/4/8 (rows 32768/G of the 32768^3 GEMM), one
# GPU: the compute side of the strong-scaling model in DESIGN §8.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
AB_ROUNDS=2 timeout 1200 python tools/experiments/ab_shapes.py "32768,32768,32768;16384,32768,32768;8192,32768,32768;4096,32768,32768" paper_2306_11148_b200/libmoa.so > gpurun_out/perrank.jsonl 2>&1; echo "rc=$?"; cat gpurun_out/perrank.jsonl | cut -c1-400
