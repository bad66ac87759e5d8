"""Per-phase breakdown of one K1 launch at small N (round-2 review item 4): a variant
build with -DMOA_K1_PHASES (tools/build_variant.sh phases -DMOA_K1_PHASES) stamps
%globaltimer per CTA at kernel entry, after griddepcontrol.wait, at the producer's
first TMA issue, at the first slab's landing (consumer warp 0), the summed
full-barrier waits, the end of the last slab and the end of the store.

    python tools/experiments/phases.py ab/libmoa_phases.so [N,N,...]

Prints one JSON line per N: medians over CTAs (ns) of each phase and the launch span
(first entry .. last store end); also the same call's CUDA-event time (eager,
back-to-back) and CUDA-graph replay time with this build, for scale.
"""
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from inputs import inputs as I  # noqa: E402

lib = ctypes.CDLL(sys.argv[1])
# PHASES_PLAN="bm,bn,stages": time that compiled K1 config instead of the chooser's
# pick (through the binding, loaded on the same variant library)
_pp = os.environ.get("PHASES_PLAN")
if _pp:
    os.environ["MOA_LIBRARY"] = os.path.abspath(sys.argv[1])
    import paper_2306_11148_b200 as moa  # noqa: E402
lib.moa_gemm.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
lib.moa_k1_phases_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "128,256,512").split(",")]
for N in sizes:
    A = torch.empty((N, N), dtype=torch.float64, device="cuda")
    B = torch.empty_like(A)
    C = torch.empty_like(A)
    I.device_fill(A, 1, I.ID_A)
    I.device_fill(B, 1, I.ID_B)
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: lib.moa_gemm(N, N, N, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, s)  # noqa: E731
    if _pp:
        bm, bn, st = (int(x) for x in _pp.split(","))
        pl = moa.Plan(**{**moa.plan(N, N, N).__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
        f = lambda: moa.gemm_with_plan(A, B, C, pl)  # noqa: E731
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    lib.moa_k1_phases_clear()
    torch.cuda.synchronize()
    f()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 8))()
    lib.moa_k1_phases_read(buf, 1024 * 8)
    rows = [[buf[b * 8 + i] for i in range(8)] for b in range(1024)]
    rows = [r for r in rows if r[0] and r[6]]
    t0 = min(r[0] for r in rows)
    med = lambda xs: round(statistics.median(xs), 1)  # noqa: E731
    out = {"N": N, "ctas": len(rows),
           "entry_after_first_ns": med([r[0] - t0 for r in rows]),
           "pdl_wait_ns": med([r[1] - r[0] for r in rows]),
           "to_first_tma_issue_ns": med([r[2] - r[1] for r in rows]),
           "first_slab_landing_ns": med([r[3] - r[2] for r in rows]),
           "summed_full_waits_ns": med([r[4] for r in rows]),
           "first_landing_to_last_slab_ns": med([r[5] - r[3] for r in rows]),
           "store_ns": med([r[6] - r[5] for r in rows]),
           "entry_to_store_end_ns": med([r[6] - r[0] for r in rows]),
           "span_ns": max(r[6] for r in rows) - t0}
    # the same call's time with CUDA events (eager back-to-back) and graph replay
    reps = 200
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    out["eager_us"] = round(a.elapsed_time(b) / reps * 1e3, 2)
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        f2 = lambda: lib.moa_gemm(N, N, N, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0,  # noqa: E731
                                  torch.cuda.current_stream().cuda_stream)
        if _pp:
            f2 = lambda: moa.gemm_with_plan(A, B, C, pl)  # noqa: E731
        f2()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                f2()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    out["graph_us"] = round(a.elapsed_time(b) / reps * 1e3, 2)
    print(json.dumps(out), flush=True)
