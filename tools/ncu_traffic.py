#!/usr/bin/env python3
"""Collect the DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per K1
launch from the ncu --set full summaries of tools/gpu_prof_configs.sh into
profiles/ncu_k1_traffic.json, keyed "MxNxP" — the roofline "traffic" figure bench.py
reports for the launch it times (rank 0's rows at G = 1, 2, 4, 8 of configs[4], and
the sweep sizes that were captured).

    python tools/ncu_traffic.py gpurun_out/ncu_cfg_*.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.prof_configs import SHAPES  # noqa: E402

out_path = os.path.join(ROOT, "profiles", "ncu_k1_traffic.json")
table = json.load(open(out_path)) if os.path.exists(out_path) else {}
for f in sys.argv[1:]:
    cfg = os.path.basename(f)[len("ncu_cfg_"):-len(".json")]
    if cfg not in SHAPES:
        continue
    d = json.load(open(f))
    caps = [c for c in d.get("captures", []) if "k_dgemm_tma" in c.get("kernel", "")]
    if not caps:
        continue
    m, n, p, _ = SHAPES[cfg]
    table[f"{m}x{n}x{p}"] = float(caps[0]["traffic_bytes"])
    print(cfg, f"{m}x{n}x{p}", caps[0]["traffic_bytes"])
json.dump(table, open(out_path, "w"), indent=1)
