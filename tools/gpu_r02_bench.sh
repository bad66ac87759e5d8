#!/bin/bash
# Round-2 GPU pass: multi-rank bench path (one GPU, NCCL stand-in), the configs[4]
# headline bench at G = 1, the ncu launch list of a bench step, and ncu --set full of
# K1 on rank 0's rows of configs[4] at G = 1, 2, 4, 8 (the roofline "traffic" figures).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_bench_multirank_gpu.py -q -m gpu -x > gpurun_out/r02_bench_mr.log 2>&1
echo "bench multirank rc=$?"; tail -5 gpurun_out/r02_bench_mr.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_g1.json 2> gpurun_out/r02_bench_g1.err
echo "bench rc=$?"; head -c 3000 gpurun_out/r02_bench_g1.json; tail -5 gpurun_out/r02_bench_g1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > gpurun_out/r02_launches_bench.log 2>&1
echo "launches rc=$?"
bash tools/gpu_prof_configs.sh ${PROF:-l1 l2 l4 l8}
