#!/bin/bash
# One-shot latency tiles with the byte rule: full GPU suite, smoke, small-N table.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/os2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/os2_smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/os2_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/os2_gpu_all.log
timeout 600 python tools/small_n.py 64,128,192,256,320,384,448,512,640,768,1024 > gpurun_out/os2_small_n.json 2> gpurun_out/os2_small_n.err; echo "small_n rc=$?"
python - <<'PY'
import json
for d in json.load(open("gpurun_out/os2_small_n.json")):
    best = sorted((c.get('graph_us', 1e9), c['cfg'][1:]) for c in d['cfgs'])
    ch = [c.get('graph_us') for c in d['cfgs'] if c['cfg'][1:] == d['chosen'][1:]]
    print(d['N'], 'chosen', d['chosen'][1:], ch, 'best', best[:3], all(c.get('bitwise', True) for c in d['cfgs']))
PY
