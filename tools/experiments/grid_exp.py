"""Grid-size experiment for the static tile schedule at small N."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
res = []
for N in (1024, 2048, 3072):
    A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    base = moa.plan(N, N, N)
    for (bm, bn, st, grid) in [(128, 128, 6, 0), (128, 64, 4, 0), (64, 64, 4, 0), (64, 64, 4, 148), (64, 64, 4, 292)]:
        q = moa.Plan(**{**base.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": grid})
        for _ in range(5): moa.gemm_with_plan(A, B, C, q)
        torch.cuda.synchronize()
        reps = 200
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps): moa.gemm_with_plan(A, B, C, q)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        res.append({"N": N, "bm": bm, "bn": bn, "grid": grid, "frac": round(2 * N**3 / (ms / 1e3) / 1e12 / 37.0, 4)})
        print(json.dumps(res[-1]), flush=True)
