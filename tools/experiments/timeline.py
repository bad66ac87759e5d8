"""Per-piece K1 timeline (variant build from tools/experiments/timeline.patch:
warp 0 of each CTA stamps globaltimer at peek start / peek done / piece done).
Summarises where a CTA's time goes at shallow vs deep k per tile."""
import ctypes, json, os, statistics, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from inputs import inputs as I  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "ab", "libmoa_timeline.so"))
lib.moa_gemm.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_void_p]
out = np.zeros(148 * 2048, dtype=np.uint64)
cnt = np.zeros(148, dtype=np.uint32)
for (m, n, p) in [(65536, 512, 512), (16384, 1024, 1024), (4096, 4096, 4096), (8192, 8192, 8192)]:
    A = torch.empty((m, n), dtype=torch.float64, device="cuda"); B = torch.empty((n, p), dtype=torch.float64, device="cuda")
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    I.device_fill(A, 1, I.ID_A); I.device_fill(B, 1, I.ID_B)
    for _ in range(2):
        lib.moa_gemm(m, n, p, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, None)
    torch.cuda.synchronize()
    lib.moa_experiment_timeline(None, None, 1)
    lib.moa_gemm(m, n, p, A.data_ptr(), B.data_ptr(), C.data_ptr(), 0, None)
    torch.cuda.synchronize()
    lib.moa_experiment_timeline(out.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p), 0)
    rec = out.reshape(148, 512, 4).astype(np.int64)
    t_min = min(rec[c, 0, 0] for c in range(148) if cnt[c])
    t_max = max(rec[c, min(cnt[c], 512) - 1, 2] for c in range(148) if cnt[c])
    waits, pieces, per_slab_first, per_slab_rest, starts, ends = [], [], [], [], [], []
    for c in range(148):
        k = min(int(cnt[c]), 512)
        if not k:
            continue
        r = rec[c, :k]
        starts.append(r[0, 0] - t_min); ends.append(t_max - r[-1, 2])
        waits.append(int((r[:, 1] - r[:, 0]).sum()))
        pieces.append(int((r[:, 2] - r[:, 1]).sum()))
        ps = (r[:, 2] - r[:, 1]) / np.maximum(r[:, 3], 1)
        per_slab_first.append(float(ps[0])); per_slab_rest.extend(ps[1:].tolist())
    span = t_max - t_min
    print(json.dumps({"shape": [m, n, p], "span_us": round(span / 1e3, 1),
                      "pieces_per_cta": round(float(np.mean(cnt[cnt > 0])), 2),
                      "peek_wait_frac": round(sum(waits) / (len(waits) * span), 4),
                      "piece_frac": round(sum(pieces) / (len(pieces) * span), 4),
                      "start_skew_us_max": round(max(starts) / 1e3, 2), "end_idle_us_mean": round(statistics.mean(ends) / 1e3, 2),
                      "end_idle_us_max": round(max(ends) / 1e3, 2),
                      "ns_per_slab_first_piece": round(statistics.median(per_slab_first), 1),
                      "ns_per_slab_other": round(statistics.median(per_slab_rest), 1) if per_slab_rest else None}), flush=True)
    del A, B, C
