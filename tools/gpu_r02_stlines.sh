#!/bin/bash
# K1 tile stores as whole 128-B row segments (lane-pair shuffle; variant
# -DMOA_K1_STORE_LINES) vs the product; bits compared across builds.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
AB_ROUNDS=5 timeout 1800 python tools/experiments/ab_shapes.py "65536,512,512;16384,1024,1024;8192,8192,8192;4096,4096,4096;2048,2048,2048;1024,1024,1024;256,256,256;300,200,260;2000,48,2000" paper_2306_11148_b200/libmoa.so ab/libmoa_stlines.so > gpurun_out/stlines_ab.jsonl 2>&1; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/stlines_ab.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list)); bits = collections.defaultdict(set)
for r in rows:
    if "error" in r: print(r); continue
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
    for k, v in r.get("bits", {}).items(): bits[k].add(v)
for k, d in agg.items():
    print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()}, "bits_identical" if len(bits[k]) == 1 else "BITS DIFFER")
PY
