#!/bin/bash
# K1 round-2 changes: static schedule + wave gate, lagged consumer groups. Parity
# first; then A/B of the schedules (tools/experiments/wave_gate.py), lag vs
# ab/libmoa_nolag.so, ncu DRAM bytes per schedule, small-N and the phase breakdown.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/r02_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_max_sizes_gpu.py tests/test_graph_capture_gpu.py tests/test_fused_gather.py tests/test_cold_launch_gpu.py -x -q > gpurun_out/r02_k1_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -3 gpurun_out/r02_k1_parity.log
[ $rc -ne 0 ] && exit 1
MOA_K1_SCHED=dynamic timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/r02_k1_parity_dyn.log 2>&1; echo "parity dyn rc=$?"; tail -1 gpurun_out/r02_k1_parity_dyn.log
timeout 1500 python tools/experiments/wave_gate.py 4096,8192,16384,32768 2 > gpurun_out/r02_wave_gate.jsonl 2>&1; echo "wg rc=$?"; cat gpurun_out/r02_wave_gate.jsonl
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "65536,512,512;16384,1024,1024;1024,1024,1024;2048,2048,2048;4096,4096,4096;8192,8192,8192" ab/libmoa_nolag.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_lag.jsonl 2>&1; echo "ab rc=$?"; cat gpurun_out/r02_ab_lag.jsonl
WG_NCU=1 timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_dgemm_tma --csv --log-file gpurun_out/r02_wave_gate_ncu.csv python tools/experiments/wave_gate.py 8192,16384,32768 1 > gpurun_out/r02_wave_gate_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python tools/small_n.py 128,256,384,512,768,1024 > gpurun_out/r02_small_n.json 2> gpurun_out/r02_small_n.err; echo "small_n rc=$?"
timeout 300 python tools/experiments/phases.py ab/libmoa_phases.so 128,256,512,1024 > gpurun_out/r02_phases.jsonl 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_phases.jsonl
