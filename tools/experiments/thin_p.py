import sys, dataclasses, json; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch, paper_2306_11148_b200 as moa
from inputs import inputs as I
from small_n import time_graph
for (m, n, p) in [(16384, 64, 32), (16384, 512, 32), (16384, 4096, 32), (12000, 256, 20), (30000, 128, 32), (1 << 20, 32, 32), (9000, 1000, 30), (256, 256, 256), (768, 768, 768), (1024, 1024, 1024)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda"); B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    ref = moa.gemm(A, B).clone(); pl = moa.plan(m, n, p)
    t = time_graph(lambda: moa.gemm(A, B, out=C), 50)
    best = []
    for (bm, bn, st) in [(64, 32, 4), (16, 32, 4), (128, 64, 4), (64, 64, 4)]:
        q = dataclasses.replace(pl, bm=bm, bn=bn, stages=st, grid=0)
        D = torch.full_like(C, float("nan")); moa.gemm_with_plan(A, B, D, q); torch.cuda.synchronize()
        assert torch.equal(D, ref)
        best.append((round(time_graph(lambda: moa.gemm_with_plan(A, B, D, q), 50) * 1e3, 2), [bm, bn]))
    print(json.dumps({"shape": [m, n, p], "chooser": [pl.bm, pl.bn], "us": round(t * 1e3, 2), "best": min(best)}))
