#!/usr/bin/env python3
"""One fp64 GEMM at N with tile (bm,bn,stages) after warm-ups, for ncu (-s 3 -c 1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N, bm, bn, st = (int(x) for x in sys.argv[1:5])
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty_like(A)
C = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
q = moa.Plan(**{**moa.plan(N, N, N).__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
for _ in range(5):
    moa.gemm_with_plan(A, B, C, q)
torch.cuda.synchronize()
