#!/bin/bash
# Bench repeatability with the final code: two more driver-contract lines back to back.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
: > gpurun_out/rep_bench.jsonl
for i in 1 2; do timeout 1500 python bench.py --no-cpu >> gpurun_out/rep_bench.jsonl 2> gpurun_out/rep_bench$i.err; echo "bench$i rc=$?"; done
python - <<'PY'
import json
for l in open("gpurun_out/rep_bench.jsonl"):
    if l.startswith("{"):
        d = json.loads(l); print(d["value"], d["roofline"]["frac"], d["energy"]["j_per_gemm"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
