"""K1 rasterisation group (tile-rows per group) at 8192^3 and 16384^3: device time
(CUDA events) for groups 4, 8, 12, 16, 24; run under ncu with --metrics
dram__bytes_read.sum,dram__bytes_write.sum for the DRAM traffic of each."""
import dataclasses
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

reps = int(os.environ.get("REPS", "5"))
for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "8192").split(",")]:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    C = torch.empty_like(A)
    ref = moa.gemm(A, B)
    base = moa.plan(N, N, N)
    for g in (4, 8, 12, 16, 24):
        pl = dataclasses.replace(base, raster_group=g)
        moa.gemm_with_plan(A, B, C, pl)
        torch.cuda.synchronize()
        ok = bool(torch.equal(C, ref))
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            moa.gemm_with_plan(A, B, C, pl)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(json.dumps({"N": N, "raster_group": g, "ms": round(statistics.median(ts), 4), "bitwise": ok}), flush=True)
    del A, B, C, ref
