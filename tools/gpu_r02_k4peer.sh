#!/bin/bash
# 3xTF32 (K4) fused-gather epilogue: scatter tests, multi-rank lifted gather through the
# NCCL stand-in, the fp32 suite, and a K4 timing check (the epilogue loop must cost nothing
# without destinations).
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1800 python -m pytest tests/test_fused_gather.py tests/test_lifted_multiproc_gpu.py tests/test_sgemm_gpu.py tests/test_lifted.py tests/test_graph_capture_gpu.py -q -x -rf > gpurun_out/k4peer_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/k4peer_tests.log
AB_DTYPE=2 AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "16384,16384,16384;8192,8192,8192" paper_2306_11148_b200/libmoa.so ab/libmoa_prepipe.so > gpurun_out/k4peer_ab.jsonl 2>&1; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/k4peer_ab.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list)); bits = collections.defaultdict(set)
for r in rows:
    if "error" in r: print(r); continue
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
    for k, v in r.get("bits", {}).items(): bits[k].add(v)
for k, d in agg.items():
    print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()}, "bits_identical" if len(bits[k]) == 1 else "BITS DIFFER")
PY
