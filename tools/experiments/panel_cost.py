"""Compute-side cost of splitting the lifted GEMM into K k-panels (the pipelined
broadcast of B, NEXT-1 step 1): moa_gemm_lifted_ex on a 1-rank NCCL communicator
(the broadcast is skipped, the K accumulate launches run) at the bench shape, CUDA
events, K = 1, 2, 4, 8; bitwise check against K = 1."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29531")
dist.init_process_group("gloo", rank=0, world_size=1)
comm = moa.Comm(device=0)
for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192,16384").split(",")]:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    C = torch.empty_like(A)
    ref = moa.gemm(A, B)
    reps = 10 if N <= 8192 else 3
    for K in (1, 2, 4, 8):
        moa.gemm_lifted(N, A, B, C, comm, npanels=K)
        torch.cuda.synchronize()
        ok = bool(torch.equal(C, ref))
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                moa.gemm_lifted(N, A, B, C, comm, npanels=K)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / reps)
        print(json.dumps({"N": N, "npanels": K, "ms": round(statistics.median(ts), 4), "bitwise": ok}), flush=True)
    del A, B, C, ref
comm.close()
