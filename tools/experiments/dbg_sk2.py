#!/usr/bin/env python3
"""For wrong elements of a stream-K run, find the k-slab range [a, b) whose partial sum
equals the wrong value (identifies stale/overwritten partials)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N, bm, bn, st, reps = (int(x) for x in sys.argv[1:6])
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
ref = A @ B
pl = moa.plan(N, N, N)
q = moa.Plan(**{**pl.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
K = -(-N // 16)
for r in range(reps):
    C = torch.full((N, N), float("nan"), dtype=torch.float64, device="cuda")
    moa.gemm_with_plan(A, B, C, q)
    torch.cuda.synchronize()
    d = (C - ref).abs()
    bad = (~(d <= 1e-9 * ref.abs().max())).nonzero()
    print(f"rep {r}: bad {len(bad)}", flush=True)
    for i, j in bad[:: max(1, len(bad) // 6)][:6].tolist():
        prod = A[i, :] * B[:, j]  # k terms
        slab = torch.stack([prod[16 * s:16 * s + 16].sum() for s in range(K)])
        cs = torch.cat([torch.zeros(1, dtype=slab.dtype, device=slab.device), slab.cumsum(0)])
        w = float(C[i, j])
        best = None
        for a in range(K + 1):
            diff = (cs[a + 1:] - cs[a] - w).abs() if a < K else None
            if diff is None:
                continue
            b = int(diff.argmin())
            e = float(diff[b])
            if best is None or e < best[0]:
                best = (e, a, a + 1 + b)
        print(f"  C[{i},{j}] tile ({i // bm},{j // bn}) wrong {w:.6f} ref {float(ref[i, j]):.6f}"
              f" ~ sum slabs [{best[1]},{best[2]}) err {best[0]:.2e}  (K={K})", flush=True)
