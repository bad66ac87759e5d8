#!/bin/bash
# One-shot latency tiles (16 stages, all of k <= 256 resident): parity (every K1 config,
# the ~300-shape sweep, fused-gather epilogue, graph capture), then graph-timed A/B of
# the chooser's pick vs the session-start build (3 alternating rounds), and the full
# small-N table (every compiled tile) for the chooser evidence.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gemm_gpu.py tests/test_shape_sweep_gpu.py tests/test_fused_gather.py tests/test_graph_capture_gpu.py -q -x > gpurun_out/os_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -3 gpurun_out/os_parity.log; [ $rc -ne 0 ] && exit 1
: > gpurun_out/os_ab.jsonl
for r in 1 2 3; do
  for lib in paper_2306_11148_b200/libmoa.so ab/libmoa_head.so; do
    MOA_LIBRARY=$PWD/$lib timeout 300 python tools/small_n.py 64,128,192,256,320,384,448,512 > gpurun_out/os_tmp.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/os_tmp.json'))
for row in d:
    ch=row['chosen']; c=[x for x in row['cfgs'] if x['cfg']==ch]
    print(json.dumps({'lib':'$lib','round':$r,'N':row['N'],'chosen':ch,'graph_us':c[0]['graph_us'] if c else None,'eager_us':c[0]['eager_us'] if c else None}))
" >> gpurun_out/os_ab.jsonl
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list); ch = {}
for l in open("gpurun_out/os_ab.jsonl"):
    r = json.loads(l); d[(r["N"], r["lib"])].append(r["graph_us"]); ch[(r["N"], r["lib"])] = r["chosen"]
for k in sorted(d): print(k, ch[k][1:], sorted(d[k])[len(d[k])//2], d[k])
PY
timeout 600 python tools/small_n.py 64,128,192,256,320,384,448,512,640,768,1024 > gpurun_out/os_small_n.json 2> gpurun_out/os_small_n.err; echo "small_n rc=$?"
python - <<'PY'
import json
for d in json.load(open("gpurun_out/os_small_n.json")):
    best = sorted((c.get('graph_us', 1e9), c['cfg'][1:]) for c in d['cfgs'])
    ch = [c.get('graph_us') for c in d['cfgs'] if c['cfg'][1:] == d['chosen'][1:]]
    print(d['N'], 'chosen', d['chosen'][1:], ch, 'best', best[:3], all(c.get('bitwise', True) for c in d['cfgs']))
PY
