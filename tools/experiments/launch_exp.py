"""Eager vs CUDA-graph-replayed timing of small GEMMs (is configs[0] launch-bound?)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
for N in (256, 512, 1024):
    A = torch.empty((N, N), dtype=torch.float64, device="cuda"); B = torch.empty_like(A); C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(10): moa.gemm(A, B, out=C)
    torch.cuda.synchronize()
    reps = 2000
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for _ in range(reps): moa.gemm(A, B, out=C)
    host_us = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record()
        for _ in range(reps): moa.gemm(A, B, out=C)
        b.record()
    torch.cuda.synchronize()
    eager_us = a.elapsed_time(b) / reps * 1e3
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(100): moa.gemm(A, B, out=C)
    with torch.cuda.stream(s):
        g.replay()
        torch.cuda.synchronize()
        a.record()
        for _ in range(20): g.replay()
        b.record()
    torch.cuda.synchronize()
    graph_us = a.elapsed_time(b) / 2000 * 1e3
    print(json.dumps({"N": N, "host_us_per_call": round(host_us, 2), "eager_us": round(eager_us, 2),
                      "graph_us": round(graph_us, 2), "graph_tflops": round(2 * N**3 / (graph_us * 1e-6) / 1e12, 3)}))
