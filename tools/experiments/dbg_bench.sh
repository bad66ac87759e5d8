mkdir -p gpurun_out
timeout 900 python -X faulthandler bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dgemm_tma -s 2 -c 1 -o gpurun_out/prof_k1_8192 \
     python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e > gpurun_out/ncu_full.log 2>&1
