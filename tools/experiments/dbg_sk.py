#!/usr/bin/env python3
"""Stream-K debug: run one config repeatedly, compare with a cuBLAS fp64 reference and
with its own first run; report mismatching tiles (tile row/col, count, max |diff|)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2306_11148_b200 as moa  # noqa: E402
from inputs import inputs as I  # noqa: E402

N, bm, bn, st, reps = (int(x) for x in sys.argv[1:6])
acc = len(sys.argv) > 6 and sys.argv[6] == "acc"
grid = int(sys.argv[7]) if len(sys.argv) > 7 else 0
A = torch.empty((N, N), dtype=torch.float64, device="cuda")
B = torch.empty_like(A)
I.device_fill(A, 1, I.ID_A)
I.device_fill(B, 1, I.ID_B)
ref = A @ B
pl = moa.plan(N, N, N)
q = moa.Plan(**{**pl.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": grid})
K = -(-N // 16)
tm_n, tn_n = -(-N // bm), -(-N // bn)
T = tm_n * tn_n
G = grid if grid else None
group = min(tm_n, 8)


def tile_id(tm, tn):  # inverse of tile_coords
    g = tm // group
    first = g * group
    gm = min(group, tm_n - first)
    return g * group * tn_n + tn * gm + (tm - first)


def label(t, G):
    dpw = T // G if T % G == 0 else (T // G - 1 if T >= 2 * G else 0)
    skf = dpw * G
    if t < skf:
        return f"dp cta {t % G}"
    U = (T - skf) * K
    lo, hi = (t - skf) * K, (t - skf + 1) * K
    owners = [c for c in range(G) if U * c // G < hi and U * (c + 1) // G > lo]
    return ("whole" if len(owners) == 1 else "split") + f" ctas {owners} " + str(
        [(U * c // G, U * (c + 1) // G) for c in owners]) + f" t={t} lo={lo}"


first = None
for r in range(reps):
    C = torch.full((N, N), float("nan"), dtype=torch.float64, device="cuda")
    if acc:
        k1 = 48
        moa.gemm_acc(A[:, :k1], B[:k1], C, accumulate=False)
        moa.gemm_acc(A[:, k1:], B[k1:], C, accumulate=True)
    else:
        moa.gemm_with_plan(A, B, C, q)
    torch.cuda.synchronize()
    d = (C - ref).abs()
    bad = ~(d <= 1e-9 * ref.abs().max())
    if first is None:
        first = C.clone()
    same = torch.equal(C, first)
    nb = int(bad.sum())
    print(f"rep {r}: bad {nb} same_as_first {same}", flush=True)
    if nb:
        idx = bad.nonzero()
        tiles = {}
        for i, j in idx.tolist():
            k = (i // bm, j // bn)
            tiles.setdefault(k, [0, 0.0])
            tiles[k][0] += 1
            tiles[k][1] = max(tiles[k][1], float(d[i, j]))
        print("  tiles:", sorted(tiles.items())[:20], "ntiles", len(tiles), flush=True)
        if G:
            kinds = {}
            for (tm, tn) in tiles:
                k = label(tile_id(tm, tn), G).split()[0]
                kinds[k] = kinds.get(k, 0) + 1
            print("  bad tiles by kind:", kinds, flush=True)
            # do bad values equal the reference (final) value of some other tile at the same in-tile offset?
            R = ref.reshape(tm_n, bm, tn_n, bn)
            for (i, j) in idx[:: max(1, len(idx) // 5)][:5].tolist():
                w = C[i, j]
                hit = ((R[:, i % bm, :, j % bn] - w).abs() < 1e-9).nonzero().tolist()
                print(f"   bad C[{i},{j}] tile ({i // bm},{j // bn}) equals ref of tiles {hit[:4]}", flush=True)
            for (tm, tn), v in sorted(tiles.items())[:4]:
                print(f"   ({tm},{tn}) n={v[0]} {label(tile_id(tm, tn), G)}", flush=True)
        ii = idx[:, 0] % bm
        jj = idx[:, 1] % bn
        print("  rows-in-tile hist", torch.bincount(ii, minlength=bm).tolist()[:bm], flush=True)
        print("  cols-in-tile hist", torch.bincount(jj, minlength=bn).tolist()[:bn], flush=True)
print("plan grid", moa.plan(N, N, N).grid, "tiles", -(-N // bm) * -(-N // bn))
