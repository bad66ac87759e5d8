import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
cases = []
for (m, n, p) in [(1984, 256, 2048), (4000, 256, 2048)]:
    A = I.host_matrix(m, n, 9, I.ID_A); B = I.host_matrix(n, p, 9, I.ID_B)
    cases.append((torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.from_numpy(O.ip(A, B, fused=True)).cuda()))
fails = collections.Counter(); total = collections.Counter()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    for ci, (tA, tB, ref) in enumerate(cases):
        for r in range(5):
            C = torch.full(ref.shape, float("nan"), dtype=torch.float64, device="cuda")
            moa.gemm(tA, tB, out=C)
            torch.cuda.synchronize()
            total[ci] += 1
            if not torch.equal(C, ref):
                fails[ci] += 1
                bad = (C != ref) | torch.isnan(C)
                nb, nn = int(bad.sum()), int(torch.isnan(C).sum())
                if fails[ci] <= 3:
                    idx = bad.nonzero()[:3].tolist()
                    print(f"case {ci} it {it} r {r}: bad {nb} nan {nn} first {idx}", flush=True)
print("env", os.environ.get("MOA_STATIC_TILES", "dynamic"), dict(fails), dict(total), flush=True)
