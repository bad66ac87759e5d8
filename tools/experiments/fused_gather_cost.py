"""Cost of the fused-gather epilogue (K1 PEER) on one GPU: moa_gemm vs
moa_gemm_scatter with 1 and 7 extra destinations (local buffers standing in for the
peers' C_full: at G = 8 each rank stores its C rows to 7 peers), and the unfused
alternative GEMM + 7 device copies of C. CUDA events, warm-up, median of windows."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402


def timeit(fn, reps, windows=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(windows):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return statistics.median(out)


def main():
    dev = torch.device("cuda:0")
    res = []
    for N in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4096,8192").split(",")]:
        A = torch.empty((N, N), dtype=torch.float64, device=dev)
        B = torch.empty((N, N), dtype=torch.float64, device=dev)
        I.device_fill(A, 1, I.ID_A)
        I.device_fill(B, 1, I.ID_B)
        C = torch.empty_like(A)
        dst = [torch.empty_like(A) for _ in range(7)]
        reps = max(3, int(0.5 / (2.0 * N ** 3 / 36e12)))
        t0 = timeit(lambda: moa.gemm(A, B, out=C), reps)
        t1 = timeit(lambda: moa.gemm_scatter(A, B, C, dst[:1]), reps)
        t7 = timeit(lambda: moa.gemm_scatter(A, B, C, dst), reps)

        def unfused():
            moa.gemm(A, B, out=C)
            for d in dst:
                d.copy_(C)
        tu = timeit(unfused, reps)
        moa.gemm_scatter(A, B, C, dst)
        torch.cuda.synchronize()
        ok = all(torch.equal(d, C) for d in dst) and torch.equal(C, moa.gemm(A, B))
        rec = {"N": N, "gemm_ms": round(t0, 4), "scatter1_ms": round(t1, 4), "scatter7_ms": round(t7, 4),
               "gemm_plus_7_copies_ms": round(tu, 4), "scatter1_overhead": round(t1 / t0 - 1, 4),
               "scatter7_overhead": round(t7 / t0 - 1, 4), "unfused7_overhead": round(tu / t0 - 1, 4),
               "bitwise": ok}
        print(json.dumps(rec), flush=True)
        res.append(rec)
        del A, B, C, dst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
