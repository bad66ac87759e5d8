#!/bin/bash
# K3 A/B: two k-slabs per ring stage (KS=2) and a producer warpgroup
# with setmaxnreg (WG), against the current build and the session-start build; plus K1
# with the wave gate off at shallow k. Bits compared across builds (checksums).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
AB_DTYPE=1 AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "16384,16384,16384;8192,8192,8192;4096,4096,4096" ab/libmoa_head.so paper_2306_11148_b200/libmoa.so ab/libmoa_k3ks2.so ab/libmoa_k3wg.so ab/libmoa_k3ks2wg.so > gpurun_out/k3ab.jsonl 2>&1; echo "k3ab rc=$?"
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "65536,512,512;16384,1024,1024;65536,1024,512;8192,8192,8192" paper_2306_11148_b200/libmoa.so paper_2306_11148_b200/libmoa.so@MOA_K1_WAVE_GATE=0 > gpurun_out/gateab.jsonl 2>&1; echo "gateab rc=$?"
python - <<'PY'
import json, collections
for f in ["gpurun_out/k3ab.jsonl", "gpurun_out/gateab.jsonl"]:
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    agg = collections.defaultdict(lambda: collections.defaultdict(list)); bits = collections.defaultdict(set)
    for r in rows:
        if "error" in r: print(r); continue
        for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
        for k, v in r.get("bits", {}).items(): bits[k].add(v)
    for k, d in agg.items():
        print(f, k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()}, "bits_identical" if len(bits[k]) == 1 else "BITS DIFFER")
PY
