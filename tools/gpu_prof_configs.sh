#!/bin/bash
# ncu --set full of the product kernel at each BASELINE config (one capture each),
# summarised by tools/ncu_summary.py into gpurun_out/ncu_cfg_<c>.json.
mkdir -p gpurun_out
declare -A FLOPS=( [c0]=33554432 [c3]=34359738368 [c16k]=8796093022208 [f32]=8796093022208 [tf32]=8796093022208 )
declare -A KERN=( [c0]=k_dgemm_tma [c3]=k_dgemm_tma [c16k]=k_dgemm_tma [f32]=k_sgemm_ffma [tf32]=k_sgemm_3xtf32 [had]=k_hadamard [kron]=k_kron )
declare -A BYTES=( [c0]=1572864 [c3]=270532608 [c16k]=6442450944 [f32]=3221225472 [tf32]=3221225472 [had]=6442450944 [kron]=2147745792 )
for c in ${@:-c0 c3 c16k f32 tf32 had kron}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KERN[$c]}" -s 1 -c 1 -o gpurun_out/prof_cfg_$c \
     python tools/prof_configs.py $c > gpurun_out/ncu_cfg_$c.log 2>&1
  echo "$c rc=$?"
  args=""
  [ -n "${FLOPS[$c]}" ] && args="$args --flops ${FLOPS[$c]}"
  [ -n "${BYTES[$c]}" ] && args="$args --bytes ${BYTES[$c]}"
  python tools/ncu_summary.py full gpurun_out/prof_cfg_$c.ncu-rep $args > gpurun_out/ncu_cfg_$c.json 2>> gpurun_out/ncu_cfg_$c.log
done
