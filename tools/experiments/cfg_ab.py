"""Same-process A/B of compiled K1 tile configs on fp64 shapes: explicit plans through
gemm_with_plan, alternating configs over R rounds (CUDA events, ~0.3 s per sample),
median TF/s per (shape, config); every config must give the same bits.

    python tools/experiments/cfg_ab.py "m,n,p;..." "bm,bn,stages[,grid];..." [ROUNDS]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1].split(";") if s]
cfgs = [tuple(int(x) for x in s.split(",")) for s in sys.argv[2].split(";") if s]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
for (m, n, p) in shapes:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    ref = moa.gemm(A, B)
    base = moa.plan(m, n, p)
    res = {c: [] for c in cfgs}
    same = {}
    for r in range(rounds):
        for c in cfgs:
            # an optional 4th entry caps the grid (moa_gemm_with_plan honours a smaller grid)
            pl = moa.Plan(**{**base.__dict__, "bm": c[0], "bn": c[1], "stages": c[2], "grid": c[3] if len(c) > 3 else 0})
            f = lambda: moa.gemm_with_plan(A, B, C, pl)  # noqa: E731
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            reps = max(3, int(300 / max(a.elapsed_time(b), 1e-3)))
            a.record()
            for _ in range(reps):
                f()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            res[c].append(2.0 * m * n * p / ms / 1e9)
            same[c] = bool(torch.equal(C, ref))
    print(json.dumps({"shape": [m, n, p], "chooser": [base.bm, base.bn, base.stages],
                      "tflops": {",".join(map(str, c)): round(statistics.median(v), 3) for c, v in res.items()},
                      "bitwise": same and all(same.values())}), flush=True)
    del A, B, C, ref
    torch.cuda.empty_cache()
