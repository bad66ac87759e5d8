"""Replica of moa_gemm_host's pipelined schedule with events on every stream, to see
where the end-to-end time goes (debug tool; the library schedule is in moa_host.cpp)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2306_11148_b200 as moa

def run(N=8192, rows0=4096, KB=8, per_rows=2048, slices=True, last_rows=0):
    m = n = p = N
    hA = torch.randn(m, n, dtype=torch.float64).pin_memory(); hB = torch.randn(n, p, dtype=torch.float64).pin_memory()
    hC = torch.empty(m, p, dtype=torch.float64).pin_memory()
    dA = torch.empty(m, n, dtype=torch.float64, device="cuda"); dB = torch.empty(n, p, dtype=torch.float64, device="cuda")
    dC = torch.empty(m, p, dtype=torch.float64, device="cuda")
    h2d, d2h, s = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
    E = lambda: torch.cuda.Event(enable_timing=True)
    marks = []
    def mark(name, stream):
        e = E(); e.record(stream); marks.append((name, e))
    bnd = [0, rows0] + list(range(rows0 + per_rows, m - last_rows, per_rows)) + ([m - last_rows] if last_rows else []) + [m]
    bnd = sorted(set(bnd))
    kb = [(n * j // KB) // 32 * 32 for j in range(KB)] + [n]
    for rep in range(2):
        marks.clear()
        torch.cuda.synchronize()
        mark("start", s)
        h2d.wait_stream(s); d2h.wait_stream(s)
        evB = []
        with torch.cuda.stream(h2d):
            if not slices:
                dA[:rows0].copy_(hA[:rows0], non_blocking=True)
            for j in range(KB):
                if slices:
                    dA[:rows0, kb[j]:kb[j + 1]].copy_(hA[:rows0, kb[j]:kb[j + 1]], non_blocking=True)
                dB[kb[j]:kb[j + 1]].copy_(hB[kb[j]:kb[j + 1]], non_blocking=True)
                e = torch.cuda.Event(); e.record(h2d); evB.append(e); mark(f"h2d B{j}", h2d)
            evA = [None]
            for i in range(1, len(bnd) - 1):
                dA[bnd[i]:bnd[i + 1]].copy_(hA[bnd[i]:bnd[i + 1]], non_blocking=True)
                e = torch.cuda.Event(); e.record(h2d); evA.append(e); mark(f"h2d A{i}", h2d)
        for i in range(len(bnd) - 1):
            if i == 0:
                for j in range(KB):
                    s.wait_event(evB[j])
                    moa.gemm_acc(dA[:rows0, kb[j]:kb[j + 1]], dB[kb[j]:kb[j + 1]], dC[:rows0], accumulate=j > 0)
                    mark(f"gemm0.{j}", s)
            else:
                s.wait_event(evA[i])
                moa.gemm(dA[bnd[i]:bnd[i + 1]], dB, out=dC[bnd[i]:bnd[i + 1]])
                mark(f"gemm{i}", s)
            e = torch.cuda.Event(); e.record(s); d2h.wait_event(e)
            with torch.cuda.stream(d2h):
                hC[bnd[i]:bnd[i + 1]].copy_(dC[bnd[i]:bnd[i + 1]], non_blocking=True)
            mark(f"d2h C{i}", d2h)
        torch.cuda.synchronize()
    t0 = marks[0][1]
    return [(n_, round(t0.elapsed_time(e), 2)) for n_, e in marks]

cfgs = []
for rows0 in (1536, 2048, 3072):
    for KB in (4, 8):
        for per_rows in (1024, 2048):
            cfgs.append(dict(rows0=rows0, KB=KB, per_rows=per_rows, slices=False, last_rows=512))
cfgs.append(dict(rows0=3072, KB=8, per_rows=2048, slices=False, last_rows=0))
for cfg in cfgs:
    tl = run(**cfg)
    print(json.dumps({"cfg": cfg, "total_ms": tl[-1][1], "timeline": tl}), flush=True)
