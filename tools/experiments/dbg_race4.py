import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
shapes = [(1984, 256, 2048), (4000, 256, 2048), (2048, 2048, 2048)]
data = []
for (m, n, p) in shapes:
    A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
    data.append((torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.from_numpy(O.ip(A, B, fused=True)).cuda()))
fails = collections.Counter()
for outer in range(int(sys.argv[1])):
    for si, (tA, tB, ref) in enumerate(data):
        for rep in range(20):
            C = moa.gemm(tA, tB)
            torch.cuda.synchronize()
            if not torch.equal(C, ref):
                fails[si] += 1
                bad = (C != ref).nonzero()
                pl = moa.plan(*shapes[si])
                tl = collections.Counter((int(r) // pl.bm, int(c) // pl.bn) for r, c in bad.tolist())
                print(f"outer {outer} shape {si} rep {rep}: bad {bad.shape[0]} tiles {dict(tl)}", flush=True)
            del C
print("env", os.environ.get("MOA_STATIC_TILES", "dynamic"), "fails", dict(fails), flush=True)
