#!/bin/bash
# small_n timing for the product and the no-fence A/B build
python tools/small_n.py 1024,2048,4096,8192,16384 > gpurun_out/small_n8_prod.json
cp paper_2306_11148_b200/libmoa.so /tmp/libmoa_prod.so
cp ab/libmoa_nofence.so paper_2306_11148_b200/libmoa.so
python tools/small_n.py 1024,2048,4096,8192,16384 > gpurun_out/small_n8_nofence.json
cp /tmp/libmoa_prod.so paper_2306_11148_b200/libmoa.so
