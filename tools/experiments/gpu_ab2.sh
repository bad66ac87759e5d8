#!/bin/bash
mkdir -p gpurun_out
python tools/experiments/ab_bench.py ab/libmoa_static.so paper_2306_11148_b200/libmoa.so 2>&1 | head -2
MOA_STATIC_TILES=1 python tools/experiments/ab_bench.py paper_2306_11148_b200/libmoa.so 2>&1 | head -1 | sed 's/^/forced-static /'
