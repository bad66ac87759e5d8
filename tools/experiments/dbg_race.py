import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
for (m, n, p) in [(1984, 256, 2048), (4000, 256, 2048), (2048, 2048, 2048)]:
    A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
    ref = torch.from_numpy(O.ip(A, B, fused=True)).cuda()
    tA, tB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    pl = moa.plan(m, n, p)
    fails = 0
    for rep in range(50):
        C = moa.gemm(tA, tB)
        torch.cuda.synchronize()
        if not torch.equal(C, ref):
            fails += 1
            if fails == 1:
                bad = (C != ref).nonzero()
                print("   first failing rep", rep, "bad", bad.shape[0], bad[:4].tolist())
    print((m, n, p), (pl.bm, pl.bn, pl.grid, pl.tiles), "env static" if os.environ.get("MOA_STATIC_TILES") else "dynamic", "fails", fails, "/ 50")
