"""Small-N fp64: every K1 tile config at its default grid vs a one-CTA-per-SM grid
(148), which turns a one-wave-but-unbalanced tile set into static stream-K runs
(tiles > grid). CUDA-graph timing (device time of back-to-back launches), bitwise
check against the default moa_gemm. One JSON line per (N, tile, grid)."""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402
from small_n import time_graph  # noqa: E402

CFGS = [(128, 128, 6), (128, 64, 4), (64, 64, 4), (64, 32, 4)]
for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "640,768,1024,1280,1536,2048").split(",")]:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    ref = moa.gemm(A, B)
    base = moa.plan(N, N, N)
    reps = max(20, int(0.3 / (2.0 * N ** 3 / 30e12)))
    t_def = time_graph(lambda: moa.gemm(A, B, out=C0), reps) if (C0 := torch.empty_like(A)) is not None else 0
    print(json.dumps({"N": N, "chooser": [base.bm, base.bn, base.grid], "us": round(t_def * 1e3, 2),
                      "frac": round(2.0 * N ** 3 / (t_def / 1e3) / 1e12 / 37.0, 4)}), flush=True)
    for (bm, bn, st) in CFGS:
        for g in (0, 148):
            pl = dataclasses.replace(base, bm=bm, bn=bn, stages=st, grid=g)
            C = torch.full_like(A, float("nan"))
            try:
                moa.gemm_with_plan(A, B, C, pl)
                torch.cuda.synchronize()
            except moa.MoAError as e:
                print(json.dumps({"N": N, "cfg": [bm, bn, st], "grid": g, "error": str(e)}), flush=True)
                continue
            ok = bool(torch.equal(C, ref))
            t = time_graph(lambda: moa.gemm_with_plan(A, B, C, pl), reps)
            print(json.dumps({"N": N, "cfg": [bm, bn, st], "grid": g or "default", "us": round(t * 1e3, 2),
                              "frac": round(2.0 * N ** 3 / (t / 1e3) / 1e12 / 37.0, 4), "bitwise": ok}), flush=True)
    del A, B, C, ref
