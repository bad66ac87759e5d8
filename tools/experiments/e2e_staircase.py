"""Replica of a 'staircase' end-to-end schedule for moa_gemm_host (research tool).

H2D order: A0, B0, A1, B1, ..., A_{KB-1}, B_{KB-1}, then the remaining A row panels.
Compute (one stream): for each B k-panel j, (a) rows [0, bnd_j) x panel j
(accumulate; the chain of every earlier block continues), (b) block j = rows
[bnd_j, bnd_{j+1}) x k [0, kb_{j+1}) in one call (a chain starting from 0, which
is bitwise the same as panel by panel). Then the remaining row panels with all of
B. C rows stream back as soon as they are final. Compared with the current
library schedule (moa.gemm_host)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402

N = 8192
m = n = p = N
hA = torch.randn(m, n, dtype=torch.float64).pin_memory()
hB = torch.randn(n, p, dtype=torch.float64).pin_memory()
hC = torch.empty(m, p, dtype=torch.float64).pin_memory()
dA = torch.empty(m, n, dtype=torch.float64, device="cuda")
dB = torch.empty(n, p, dtype=torch.float64, device="cuda")
dC = torch.empty(m, p, dtype=torch.float64, device="cuda")
h2d, d2h, s = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()


def staircase(blocks, KB=8, per_rows=2048, last_rows=512):
    bnd = [0]
    for r in blocks:
        bnd.append(bnd[-1] + r)
    R = bnd[-1]
    rest = list(range(R + per_rows, m - last_rows, per_rows)) + ([m - last_rows] if last_rows else [])
    pb = [R] + [x for x in rest if R < x < m] + [m]
    kb = [(n * j // KB) // 32 * 32 for j in range(KB)] + [n]
    ev = {}
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(s)
    h2d.wait_stream(s)
    d2h.wait_stream(s)
    with torch.cuda.stream(h2d):
        for j in range(KB):
            if j < len(blocks):
                dA[bnd[j]:bnd[j + 1]].copy_(hA[bnd[j]:bnd[j + 1]], non_blocking=True)
            dB[kb[j]:kb[j + 1]].copy_(hB[kb[j]:kb[j + 1]], non_blocking=True)
            e = torch.cuda.Event()
            e.record(h2d)
            ev[("B", j)] = e
        for i in range(len(pb) - 1):
            dA[pb[i]:pb[i + 1]].copy_(hA[pb[i]:pb[i + 1]], non_blocking=True)
            e = torch.cuda.Event()
            e.record(h2d)
            ev[("A", i)] = e
    for j in range(KB):
        s.wait_event(ev[("B", j)])
        if j > 0 and bnd[min(j, len(blocks))] > 0:
            r = bnd[min(j, len(blocks))]
            moa.gemm_acc(dA[:r, kb[j]:kb[j + 1]], dB[kb[j]:kb[j + 1]], dC[:r], accumulate=True)
        if j < len(blocks):
            moa.gemm_acc(dA[bnd[j]:bnd[j + 1], :kb[j + 1]], dB[:kb[j + 1]], dC[bnd[j]:bnd[j + 1]], accumulate=False)
    e = torch.cuda.Event()
    e.record(s)
    d2h.wait_event(e)
    with torch.cuda.stream(d2h):
        hC[:R].copy_(dC[:R], non_blocking=True)
    for i in range(len(pb) - 1):
        s.wait_event(ev[("A", i)])
        moa.gemm(dA[pb[i]:pb[i + 1]], dB, out=dC[pb[i]:pb[i + 1]])
        e = torch.cuda.Event()
        e.record(s)
        d2h.wait_event(e)
        with torch.cuda.stream(d2h):
            hC[pb[i]:pb[i + 1]].copy_(dC[pb[i]:pb[i + 1]], non_blocking=True)
    s.wait_stream(d2h)
    s1.record(s)
    torch.cuda.synchronize()
    return s0.elapsed_time(s1)


def library():
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(s)
    moa.gemm_host(hA, hB, hC, dA, dB, dC)
    s1.record(s)
    torch.cuda.synchronize()
    return s0.elapsed_time(s1)


cands = {
    "lib": None,
    "u384x8": [384] * 8,
    "u512x8": [512] * 8,
    "grow128": [128, 256, 384, 512, 640, 768, 896, 1024],
    "grow256": [256, 384, 512, 640, 768, 896, 1024, 1152],
    "front1024": [1024, 256, 256, 256, 256, 256, 256, 256],
    "front1536": [1536, 256, 256, 256, 256, 256, 256, 256],
    "u768x4_KB4": ([768] * 4, 4),
}
for rep in range(2):
    for name, c in cands.items():
        if c is None:
            t = library()
        elif isinstance(c, tuple):
            t = staircase(c[0], KB=c[1])
        else:
            t = staircase(c)
        if rep == 1:
            print(json.dumps({"name": name, "ms": round(t, 3)}), flush=True)
