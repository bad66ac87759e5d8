#!/bin/bash
# (1) smoke timing twice (a 120 s timeout hit once on a fresh box); (2) timing-only A/B:
# K1 with whole-tile stores skipped (variant -DMOA_K1_NOSTORE_EXPERIMENT, wrong results)
# vs the product at shallow and deep k: is the tile-end store burst the shallow-k loss?
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for i in 1 2; do s=$(date +%s.%N); timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ns_smoke$i.log 2>&1; rc=$?; echo "smoke$i rc=$rc $(python -c "print(round($(date +%s.%N)-$s,1))") s"; tail -1 gpurun_out/ns_smoke$i.log; done
timeout 1200 python -m pytest tests/test_gemm_gpu.py tests/test_shape_sweep_gpu.py tests/test_fused_gather.py -q -x > gpurun_out/ns_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/ns_parity.log
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "65536,512,512;16384,1024,1024;8192,8192,8192" paper_2306_11148_b200/libmoa.so ab/libmoa_nostore.so > gpurun_out/nostore_ab.jsonl 2>&1; echo "ab rc=$?"
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/nostore_ab.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "error" in r: print(r); continue
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
for k, d in agg.items(): print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()})
PY
