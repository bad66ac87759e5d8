#!/bin/bash
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gather.py tests/test_shape_sweep_gpu.py -q -x > gpurun_out/r02_parity_lat.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -2 gpurun_out/r02_parity_lat.log; [ $rc -ne 0 ] && exit 1
timeout 600 python tools/small_n.py 64,128,192,256,320,384,448,512,640,768,1024 > gpurun_out/r02_small_n_lat.json 2> gpurun_out/r02_small_n_lat.err; echo "small_n rc=$?"
python - <<'PY'
import json
for d in json.load(open("gpurun_out/r02_small_n_lat.json")):
    best = sorted((c.get('graph_us', 1e9), c['cfg'][1:]) for c in d['cfgs'])
    ch = [c.get('graph_us') for c in d['cfgs'] if c['cfg'][1:] == d['chosen'][1:]]
    print(d['N'], 'chosen', d['chosen'][1:], ch, 'best', best[:3], all(c.get('bitwise', True) for c in d['cfgs']))
PY
