"""Latency tiles (16x32) with 4 / 8 / 16-stage rings at N = 128..512 (needs the deep-ring
configs compiled in temporarily; result: no gain, profiles/r01_latency_stages.jsonl —
the chain of dependent DMMAs, not TMA latency, bounds config0)."""
import dataclasses, json, os, sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from small_n import time_graph, time_fn
for N in [128, 256, 384, 512]:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    ref = moa.gemm(A, B); base = moa.plan(N, N, N)
    for st in (4, 8, 16):
        pl = dataclasses.replace(base, bm=16, bn=32, stages=st, grid=0)
        C = torch.full_like(A, float("nan")); moa.gemm_with_plan(A, B, C, pl); torch.cuda.synchronize()
        ok = bool(torch.equal(C, ref))
        tg = time_graph(lambda: moa.gemm_with_plan(A, B, C, pl), 200)
        te = time_fn(lambda: moa.gemm_with_plan(A, B, C, pl), 200)
        print(json.dumps({"N": N, "stages": st, "graph_us": round(tg*1e3, 2), "eager_us": round(te*1e3, 2), "bitwise": ok}), flush=True)
