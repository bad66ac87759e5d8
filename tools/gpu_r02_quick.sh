#!/bin/bash
# quick: K1 parity + A/B against the round-1 build and the gate off
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_fused_gather.py tests/test_graph_capture_gpu.py -q -x > gpurun_out/r02_parity4.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -2 gpurun_out/r02_parity4.log; [ $rc -ne 0 ] && exit 1
AB_ROUNDS=3 timeout 1500 python tools/experiments/ab_shapes.py "${SHAPES:-65536,512,512;16384,1024,1024;8192,8192,8192;4096,4096,4096;2048,2048,2048;1024,1024,1024;768,768,768}" ab/libmoa_r01.so paper_2306_11148_b200/libmoa.so paper_2306_11148_b200/libmoa.so@MOA_K1_WAVE_GATE=0 > gpurun_out/r02_ab_quick.jsonl 2>&1; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/r02_ab_quick.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
for k, d in agg.items():
    print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()})
PY
