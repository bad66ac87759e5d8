"""Pinned host<->device copy bandwidths (H2D, D2H, concurrent), the inputs of the e2e schedule."""
import torch, json
G = 1 << 30
h = torch.empty(G // 8, dtype=torch.float64).pin_memory()
h2 = torch.empty(G // 8, dtype=torch.float64).pin_memory()
d = torch.empty(G // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(G // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h.copy_(d, non_blocking=True))
def both():
    e = torch.cuda.Event(); e.record()
    s1.wait_event(e); s2.wait_event(e)
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
both_ms = t(both)
print(json.dumps({"h2d_GBps": round(G / h2d / 1e6, 1), "d2h_GBps": round(G / d2h / 1e6, 1),
                  "concurrent_ms_1GiB_each_way": round(both_ms, 2), "concurrent_h2d_GBps": round(G / both_ms / 1e6, 1)}))
