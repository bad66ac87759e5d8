#!/bin/bash
# Latency tiles with a 32-bit tile map (configs[0]): parity + graph-timed A/B vs the
# session-start build, alternating builds over 3 rounds (tools/small_n.py, MOA_LIBRARY).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x -k "latency or config0 or tile_edge or each_compiled" > gpurun_out/lat_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -2 gpurun_out/lat_parity.log; [ $rc -ne 0 ] && exit 1
: > gpurun_out/lat_ab.jsonl
for r in 1 2 3; do
  for lib in paper_2306_11148_b200/libmoa.so ab/libmoa_head.so; do
    MOA_LIBRARY=$PWD/$lib timeout 300 python tools/small_n.py 128,256,384,512 > gpurun_out/lat_tmp.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/lat_tmp.json'))
for row in d:
    ch=row['chosen']; c=[x for x in row['cfgs'] if x['cfg']==ch]
    print(json.dumps({'lib':'$lib','round':$r,'N':row['N'],'chosen':ch,'graph_us':c[0]['graph_us'] if c else None,'eager_us':c[0]['eager_us'] if c else None}))
" >> gpurun_out/lat_ab.jsonl
  done
done
python - <<'PY'
import json, collections
d = collections.defaultdict(list)
for l in open("gpurun_out/lat_ab.jsonl"):
    r = json.loads(l); d[(r["N"], r["lib"])].append(r["graph_us"])
for k in sorted(d): print(k, sorted(d[k])[len(d[k])//2], d[k])
PY
