#!/bin/bash
# K5 DFMA latency tiles + K1 runtime lag + K3 lag: parity, then small-N sweep and A/Bs.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/r02_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 1500 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gather.py tests/test_graph_capture_gpu.py tests/test_sgemm_gpu.py tests/test_shape_sweep_gpu.py tests/test_max_sizes_gpu.py tests/test_lifted_multiproc_gpu.py -q -x > gpurun_out/r02_parity2.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -3 gpurun_out/r02_parity2.log
[ $rc -ne 0 ] && exit 1
timeout 900 python tools/small_n.py 64,128,192,256,384,512,768,1024 > gpurun_out/r02_small_n_k5.json 2> gpurun_out/r02_small_n_k5.err; echo "small_n rc=$?"; cat gpurun_out/r02_small_n_k5.err | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    best = sorted((c.get('graph_us', 1e9), c['cfg']) for c in d['cfgs'])
    print(d['N'], 'chosen', d['chosen'], 'best', best[:4], 'bitwise', all(c.get('bitwise', True) for c in d['cfgs']))
"
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "65536,512,512;16384,1024,1024;8192,8192,8192;2048,2048,2048" ab/libmoa_nolag.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_lag2.jsonl 2>&1; echo "ab lag rc=$?"; cat gpurun_out/r02_ab_lag2.jsonl | cut -c1-260
AB_DTYPE=1 AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "8192,8192,8192;16384,16384,16384;4096,4096,4096" ab/libmoa_k3nolag.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_k3lag.jsonl 2>&1; echo "ab k3 rc=$?"; cat gpurun_out/r02_ab_k3lag.jsonl | cut -c1-200
