#!/bin/bash
# many fresh processes: the failure showed on the first launch of an instantiation
for i in $(seq 1 12); do timeout 200 python tools/experiments/dbg_race4.py 1 2>&1 | grep -E "outer|env"; done
python tools/experiments/ab_bench.py ab/libmoa_static.so paper_2306_11148_b200/libmoa.so 2>&1 | head -2
