set -x
for c in "64 64 4" "32 32 3" "128 64 4"; do
  t=$(echo $c | tr ' ' _)
  ncu --set full --clock-control none -k regex:k_dgemm_tma -s 3 -c 1 -o gpurun_out/ncu_n1024_$t python tools/experiments/prof_small.py 1024 $c > /dev/null 2>&1
done
ls gpurun_out
