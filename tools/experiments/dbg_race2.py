import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
m, n, p = 4000, 256, 2048
A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
ref = torch.from_numpy(O.ip(A, B, fused=True)).cuda()
tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
base = moa.plan(m, n, p)
for (bm, bn, st) in [(128, 64, 4), (64, 64, 4), (128, 128, 6)]:
    q = moa.Plan(**{**base.__dict__, "bm": bm, "bn": bn, "stages": st})
    fails = 0
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    for rep in range(reps):
        C.fill_(float("nan"))
        moa.gemm_with_plan(tA, tB, C, q)
        torch.cuda.synchronize()
        if not torch.equal(C, ref):
            fails += 1
            if fails <= 2:
                bad = (C != ref).nonzero().cpu().numpy()
                tiles = collections.Counter((int(r) // bm, int(c) // bn) for r, c in bad)
                nan = int(torch.isnan(C).sum())
                print(f"  {bm}x{bn} rep {rep}: bad {len(bad)} nan {nan} tiles {dict(list(tiles.items())[:6])} rows {sorted(set(int(r) % bm for r, c in bad))[:12]} cols {sorted(set(int(c) % bn for r, c in bad))[:12]}")
    print(f"{bm}x{bn} fails {fails}/{reps}", flush=True)
