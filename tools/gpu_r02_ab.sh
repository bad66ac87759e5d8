#!/bin/bash
# generic A/B: SHAPES and LIBS from the environment (fp64 unless AB_DTYPE)
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
AB_ROUNDS=${AB_ROUNDS:-3} timeout 1500 python tools/experiments/ab_shapes.py "$SHAPES" $LIBS > gpurun_out/${OUT:-r02_ab}.jsonl 2>&1; echo "ab rc=$?"
python - <<PY
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/${OUT:-r02_ab}.jsonl") if l.startswith("{")]
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if "error" in r: print(r); continue
    for k, v in r.get("tflops", {}).items(): agg[k][r["lib"]].append(v)
for k, d in agg.items():
    print(k, {l: round(sorted(v)[len(v)//2], 3) for l, v in d.items()})
PY
