#!/bin/bash
# ncu --set full of the product kernel at each BASELINE config (one capture each),
# summarised by tools/ncu_summary.py into gpurun_out/ncu_cfg_<c>.json.
mkdir -p gpurun_out
declare -A FLOPS=( [l1]=70368744177664 [l2]=35184372088832 [l4]=17592186044416 [l8]=8796093022208 [c0]=33554432 [c3]=34359738368 [c16k]=8796093022208 [f32]=8796093022208 [tf32]=8796093022208 )
declare -A KERN=( [l1]=k_dgemm_tma [l2]=k_dgemm_tma [l4]=k_dgemm_tma [l8]=k_dgemm_tma [c0]=k_dgemm_tma [c3]=k_dgemm_tma [c16k]=k_dgemm_tma [f32]=k_sgemm_ffma [tf32]=k_sgemm_3xtf32 [had]=k_hadamard [kron]=k_kron )
declare -A BYTES=( [l1]=25769803776 [l2]=17179869184 [l4]=12884901888 [l8]=10737418240 [c0]=1572864 [c3]=270532608 [c16k]=6442450944 [f32]=3221225472 [tf32]=3221225472 [had]=6442450944 [kron]=2147745792 )
for c in ${@:-c0 c3 c16k f32 tf32 had kron}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KERN[$c]}" -s 1 -c 1 -o gpurun_out/prof_cfg_$c \
     python tools/prof_configs.py $c > gpurun_out/ncu_cfg_$c.log 2>&1
  echo "$c rc=$?"
  args=""
  [ -n "${FLOPS[$c]}" ] && args="$args --flops ${FLOPS[$c]}"
  [ -n "${BYTES[$c]}" ] && args="$args --bytes ${BYTES[$c]}"
  python tools/ncu_summary.py full gpurun_out/prof_cfg_$c.ncu-rep $args > gpurun_out/ncu_cfg_$c.json 2>> gpurun_out/ncu_cfg_$c.log
done
