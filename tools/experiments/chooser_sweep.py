"""Static chooser vs the best compiled K1 tile over a grid of fp64 shapes (tall,
wide, thin, deep). CUDA-graph device time; one JSON line per shape with the chooser's
pick, its time, the best tile and the ratio."""
import dataclasses
import itertools
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

CFGS = [(128, 128, 6), (128, 64, 4), (64, 64, 4), (64, 32, 4), (16, 32, 4), (16, 16, 4), (16, 32, 8), (16, 16, 8),
        (16, 32, 16), (16, 16, 16)]
ms = [256, 2048, 16384, 1 << 17]
ns = [64, 512, 4096]
ps = [32, 96, 200, 512, 2048, 8192]
worst = []
for m, n, p in itertools.product(ms, ns, ps):
    fl = 2.0 * m * n * p
    if fl > 2e11 or 8 * (m * n + n * p + m * p) > 3e9:
        continue
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    base = moa.plan(m, n, p)
    reps = max(3, min(200, int(0.05 / (fl / 30e12 + 5e-6))))
    t_ch = time_graph(lambda: moa.gemm(A, B, out=C), reps)
    best = (t_ch, [base.bm, base.bn])
    for (bm, bn, st) in CFGS:
        pl = dataclasses.replace(base, bm=bm, bn=bn, stages=st, grid=0)
        t = time_graph(lambda: moa.gemm_with_plan(A, B, C, pl), reps)
        best = min(best, (t, [bm, bn]))
    rec = {"shape": [m, n, p], "chooser": [base.bm, base.bn], "chooser_us": round(t_ch * 1e3, 2),
           "best": best[1], "best_us": round(best[0] * 1e3, 2), "ratio": round(t_ch / best[0], 3),
           "chooser_tfs": round(fl / t_ch / 1e9, 2)}
    print(json.dumps(rec), flush=True)
    del A, B, C
