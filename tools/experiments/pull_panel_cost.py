"""Compute-side cost of the pulled exchange's k-panel chain on one GPU (DESIGN §8
scaling model): per-rank shape of BASELINE configs[4] at G = 2/4/8 (rows 32768/G),
one moa_gemm launch vs the moa_gemm_acc chain over moa_pull_panels(n) boundaries
(what ranks g > 0 run in moa_gemm_lifted with B in a window). CUDA events, alternating,
bits compared. One JSON line per G."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N = int(os.environ.get("PPC_N", "32768"))
bnd = moa.pull_panels(N)
B = torch.empty((N, N), dtype=torch.float64, device="cuda")
I.device_fill(B, 1, I.ID_B)
for G in [int(g) for g in os.environ.get("PPC_G", "2,4,8").split(",")]:
    rows = N // G
    A = torch.empty((rows, N), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    C1 = torch.empty((rows, N), dtype=torch.float64, device="cuda")
    C2 = torch.empty((rows, N), dtype=torch.float64, device="cuda")

    def one():
        moa.gemm(A, B, out=C1)

    def chain():
        for j in range(len(bnd) - 1):
            k0, k1 = bnd[j], bnd[j + 1]
            moa.gemm_acc(A[:, k0:k1], B[k0:k1], C2, j > 0)

    t = {"one": [], "chain": []}
    one(); chain(); torch.cuda.synchronize()
    for _ in range(3):
        for name, f in (("one", one), ("chain", chain)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            t[name].append(a.elapsed_time(b))
    one_ms, chain_ms = statistics.median(t["one"]), statistics.median(t["chain"])
    print(json.dumps({"G": G, "rows": rows, "n": N, "panels": bnd, "one_ms": round(one_ms, 3),
                      "chain_ms": round(chain_ms, 3), "chain_cost": round(chain_ms / one_ms - 1, 5),
                      "bitwise": bool(torch.equal(C1, C2))}), flush=True)
    del A, C1, C2
    torch.cuda.empty_cache()
