#!/bin/bash
# product stream-K: timing + DRAM bytes at 8192/16384 (compare with profiles: dynamic 6.8 GB / 60 GB, 82% L2 hit)
python tools/small_n.py 1024,2048,4096,8192,16384 2>/dev/null > gpurun_out/ab_dyn_prod2.json
for N in 8192 16384; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:k_dgemm_tma -s 3 -c 1 --csv python tools/experiments/prof_small.py $N 128 128 6 2>/dev/null | grep -E "dram|lts|gpu__time" > gpurun_out/ab_dyn_ncu_prod2_$N.csv
done
