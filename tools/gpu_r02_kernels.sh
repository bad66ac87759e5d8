#!/bin/bash
# Round-2 GPU pass 2: full GPU suite; small-N one-shot tiles; phase breakdown (variant
# build); A/B of the st.async piece descriptors vs the previous build; sanitizers;
# J per DRAM GB (raster groups) at 16384^3 and 32768^3.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_gpu_all2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_gpu_all2.log
timeout 600 python tools/small_n.py 128,256,384,512,768,1024 > gpurun_out/r02_small_n.json 2> gpurun_out/r02_small_n.err; echo "small_n rc=$?"
timeout 300 python tools/experiments/phases.py ab/libmoa_phases.so 128,256,512 > gpurun_out/r02_phases.jsonl 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_phases.jsonl
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "256,256,256;1024,1024,1024;2048,2048,2048;4096,4096,4096;8192,8192,8192;65536,512,512" ab/libmoa_pre_desc.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_desc.jsonl 2>&1; echo "ab rc=$?"; cat gpurun_out/r02_ab_desc.jsonl
bash tools/gpu_sanitize.sh
timeout 600 python tools/experiments/energy_traffic.py 16384 1,2,4,8,16 > gpurun_out/r02_energy_traffic_16384.jsonl 2>&1; echo "energy16k rc=$?"; cat gpurun_out/r02_energy_traffic_16384.jsonl
RASTER_NCU=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dgemm_tma -s 1 --csv --log-file gpurun_out/r02_raster_ncu_16384.csv python tools/experiments/energy_traffic.py 16384 1,2,4,8,16 > /dev/null 2>&1; echo "ncu16k rc=$?"
ROUNDS=3 timeout 900 python tools/experiments/energy_traffic.py 32768 2,8,32 > gpurun_out/r02_energy_traffic_32768.jsonl 2>&1; echo "energy32k rc=$?"; cat gpurun_out/r02_energy_traffic_32768.jsonl
RASTER_NCU=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dgemm_tma -s 1 --csv --log-file gpurun_out/r02_raster_ncu_32768.csv python tools/experiments/energy_traffic.py 32768 2,8,32 > /dev/null 2>&1; echo "ncu32k rc=$?"
