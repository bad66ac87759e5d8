#!/usr/bin/env python3
"""Small-N fp64 tile experiment: every compiled K1 tile config at N = 256..4096
(and 16384 for eta), timed two ways:
  eager  — R back-to-back moa.gemm_with_plan calls (includes host submit cost)
  graph  — the same R calls captured once in a CUDA graph and replayed (device time)
Inputs resident in HBM; events on the current stream. One JSON document on stdout.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

PEAK = 37.0
CFGS = [("dgemm_tma", 128, 128, 6), ("dgemm_tma", 128, 64, 4), ("dgemm_tma", 64, 64, 4), ("dgemm_tma", 64, 32, 4),
        ("dgemm_tma", 16, 32, 4), ("dgemm_tma", 16, 16, 4), ("dgemm_tma", 16, 32, 8), ("dgemm_tma", 16, 16, 8),
        ("dgemm_tma", 16, 32, 16), ("dgemm_tma", 16, 16, 16)]


def time_fn(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def time_graph(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,384,512,768,1024,1280,1536,2048,3072,4096,16384").split(",")]
    out = []
    for N in sizes:
        A = torch.empty((N, N), dtype=torch.float64, device="cuda")
        B = torch.empty_like(A)
        C = torch.empty_like(A)
        I.device_fill(A, 1, I.ID_A)
        I.device_fill(B, 1, I.ID_B)
        ref = torch.empty_like(C)
        moa.gemm(A, B, out=ref)
        pl = moa.plan(N, N, N)
        fl = 2.0 * N ** 3
        reps = max(5, min(2000, int(0.3 / (fl / 30e12))))
        row = {"N": N, "chosen": [pl.kernel, pl.bm, pl.bn, pl.stages], "cfgs": []}
        for kern, bm, bn, st in CFGS:
            q = moa.Plan(**{**pl.__dict__, "kernel": kern, "bm": bm, "bn": bn, "stages": st, "grid": 0})
            fn = lambda: moa.gemm_with_plan(A, B, C, q)  # noqa: E731
            try:
                e = time_fn(fn, reps)
                g = time_graph(fn, min(reps, 200)) if N <= 4096 else e
            except moa.MoAError as ex:
                row["cfgs"].append({"cfg": [kern, bm, bn, st], "error": str(ex)})
                continue
            ok = torch.equal(C, ref)
            row["cfgs"].append({"cfg": [kern, bm, bn, st], "eager_us": round(e * 1e3, 2), "graph_us": round(g * 1e3, 2),
                                "frac_graph": round(fl / (g / 1e3) / 1e12 / PEAK, 4), "bitwise": ok})
        out.append(row)
        print(json.dumps(row), file=sys.stderr)
        del A, B, C, ref
        torch.cuda.empty_cache()
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
