"""True-HBM diagnostic: fp64 m = 2^20, n = p = 32 (4 flop/B) and other
thin-p shapes, every compiled K1 tile vs the chooser's pick; HBM GB/s on the
compulsory bytes 8(mn + np + mp), bitwise check against the chooser's result."""
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

CFGS = [(128, 128, 6), (128, 64, 4), (64, 64, 4), (64, 32, 4), (16, 32, 4), (16, 16, 4)]
for (m, n, p) in [(1 << 20, 32, 32), (1 << 20, 64, 64), (1 << 20, 16, 16), (1 << 18, 128, 32), (1 << 20, 96, 96)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    ref = moa.gemm(A, B)
    base = moa.plan(m, n, p)
    byts = 8.0 * (m * n + n * p + m * p)
    fl = 2.0 * m * n * p
    C = torch.empty_like(ref)
    t = time_graph(lambda: moa.gemm(A, B, out=C), 50)
    print(json.dumps({"shape": [m, n, p], "chooser": [base.bm, base.bn, base.grid], "us": round(t * 1e3, 2),
                      "GBs": round(byts / (t / 1e3) / 1e9, 1), "TFs": round(fl / (t / 1e3) / 1e12, 2)}), flush=True)
    for (bm, bn, st) in CFGS:
        pl = dataclasses.replace(base, bm=bm, bn=bn, stages=st, grid=0)
        C = torch.full_like(ref, float("nan"))
        moa.gemm_with_plan(A, B, C, pl)
        torch.cuda.synchronize()
        ok = bool(torch.equal(C, ref))
        t = time_graph(lambda: moa.gemm_with_plan(A, B, C, pl), 50)
        print(json.dumps({"shape": [m, n, p], "cfg": [bm, bn], "us": round(t * 1e3, 2),
                          "GBs": round(byts / (t / 1e3) / 1e9, 1), "TFs": round(fl / (t / 1e3) / 1e12, 2),
                          "bitwise": ok}), flush=True)
