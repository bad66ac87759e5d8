#!/bin/bash
# K1: cross-slab software pipeline of the fragment loads (next stage waited for
# and its first fragments loaded before the last k-step DMMAs): parity, then A/B vs the previous build.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gather.py -q -x > gpurun_out/pipe_parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -2 gpurun_out/pipe_parity.log; [ $rc -ne 0 ] && exit 1
AB_ROUNDS=5 timeout 1800 python tools/experiments/ab_shapes.py "${SHAPES:-8192,8192,8192;16384,16384,16384;4096,4096,4096;65536,512,512;16384,1024,1024;2048,2048,2048;1024,1024,1024}" paper_2306_11148_b200/libmoa.so ab/libmoa_prepipe.so > gpurun_out/pipe_ab.jsonl 2>&1; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/pipe_ab.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list)); bits = collections.defaultdict(set)
for r in rows:
    if "error" in r: print(r); continue
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
    for k, v in r.get("bits", {}).items(): bits[k].add(v)
for k, d in agg.items():
    print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()}, "bits_identical" if len(bits[k]) == 1 else "BITS DIFFER")
PY
