#!/usr/bin/env python3
"""Stream-K vs dynamic A/B: time every K1 tile config on square and skinny shapes
(CUDA-graph replay, inputs resident). Run once per library build; JSON on stdout."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402
from tools.small_n import time_graph, time_fn  # noqa: E402

SHAPES = [(1536, 1536, 1536), (2048, 2048, 2048), (3072, 3072, 3072), (4096, 4096, 4096), (6144, 6144, 6144),
          (8192, 8192, 8192), (65536, 512, 512), (32768, 1024, 1024), (16384, 2048, 2048), (8192, 4096, 8192)]
CFGS = [(128, 128, 6), (128, 64, 4), (64, 64, 4)]
out = []
for (m, n, p) in SHAPES:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    pl = moa.plan(m, n, p)
    fl = 2.0 * m * n * p
    row = {"shape": [m, n, p], "chosen": [pl.bm, pl.bn], "cfgs": []}
    for bm, bn, st in CFGS:
        q = moa.Plan(**{**pl.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
        fn = lambda: moa.gemm_with_plan(A, B, C, q)  # noqa: E731
        reps = max(3, min(200, int(0.2 / (fl / 30e12))))
        t = time_graph(fn, reps) if fl < 2e11 else time_fn(fn, reps)
        row["cfgs"].append({"cfg": [bm, bn], "us": round(t * 1e3, 2), "frac": round(fl / (t / 1e3) / 1e12 / 37.0, 4)})
    out.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    del A, B, C
    torch.cuda.empty_cache()
json.dump(out, sys.stdout)
