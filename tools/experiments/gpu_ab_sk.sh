#!/bin/bash
# A/B: product vs ab/libmoa_$1.so on tools/ab_sk.py shapes (product run twice to bracket drift)
cp paper_2306_11148_b200/libmoa.so /tmp/libmoa_prod.so
python tools/ab_sk.py > gpurun_out/ab_sk_prod.json 2>/dev/null
cp ab/libmoa_$1.so paper_2306_11148_b200/libmoa.so
python tools/ab_sk.py > gpurun_out/ab_sk_$1.json 2>/dev/null
cp /tmp/libmoa_prod.so paper_2306_11148_b200/libmoa.so
python tools/ab_sk.py > gpurun_out/ab_sk_prod2.json 2>/dev/null
