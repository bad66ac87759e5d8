"""Soak of the one-shot latency tiles: random tiny fp64 shapes (n <= 256, one tile per
CTA), each launched many times back to back (PDL overlap of consecutive grids) and in a
CUDA graph, every result bitwise equal to the same product through the ring-fed 16x16
tile (explicit plan). One JSON line at the end."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("SOAK_SEED", "11")))
shapes = 0
launches = 0
bad = []
oneshot = 0
for it in range(int(os.environ.get("SOAK_SHAPES", "200"))):
    m, p = (int(x) for x in rng.integers(1, 300, size=2))
    n = int(rng.integers(1, 257))
    if rng.random() < 0.6:
        n, p = n + (-n) % 2, p + (-p) % 2
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 100 + it, I.ID_A)
    I.device_fill(B, 100 + it, I.ID_B)
    pl = moa.plan(m, n, p)
    oneshot += int(pl.stages == 16)
    ref = torch.empty((m, p), dtype=torch.float64, device="cuda")
    q = moa.Plan(**{**pl.__dict__, "bm": 16, "bn": 16, "stages": 8, "grid": 0}) if pl.kernel == "dgemm_tma" else pl
    moa.gemm_with_plan(A, B, ref, q)
    outs = [torch.full((m, p), float("nan"), dtype=torch.float64, device="cuda") for _ in range(8)]
    for r in range(4):
        for o in outs:
            moa.gemm(A, B, out=o)
            launches += 1
    torch.cuda.synchronize()
    for o in outs:
        if not torch.equal(o, ref):
            bad.append([m, n, p, "eager"])
            break
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for o in outs:
                moa.gemm(A, B, out=o)
    for r in range(3):
        for o in outs:
            o.fill_(float("nan"))
        g.replay()
        launches += len(outs)
    torch.cuda.synchronize()
    for o in outs:
        if not torch.equal(o, ref):
            bad.append([m, n, p, "graph"])
            break
    shapes += 1
print(json.dumps({"shapes": shapes, "one_shot_shapes": oneshot, "launches": launches, "mismatches": bad}))
