"""Small-shape runs of every kernel (K1 fp64 TMA, K2 generic, K3 FFMA, K3g, K4 3xTF32)
for compute-sanitizer (memcheck / racecheck / synccheck), plus K1 in its stream-K
(1920x1024x1920: 225 128x128 tiles on 148 CTAs), 64x32 stream-K over 3 CTAs/SM (2000x48x2000)
and dynamic + stream-K (7040x16x7040) schedules, the one-shot latency tiles (n <= 256,
also in accumulate mode) and a ring-fed latency tile."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O
ok = True
for (m, n, p) in [(200, 96, 260), (130, 34, 66), (256, 256, 256)]:
    for dt, prec in [(np.float64, None), (np.float32, None), (np.float32, "3xtf32")]:
        A = I.host_matrix(m, n, 2, I.ID_A, dtype=dt); B = I.host_matrix(n, p, 2, I.ID_B, dtype=dt)
        C = moa.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), precision=prec)
        torch.cuda.synchronize()
        err = np.linalg.norm(C.cpu().numpy() - O.ip(A, B)) / np.linalg.norm(O.ip(A, B))
        print(m, n, p, dt.__name__, prec, moa.plan(m, n, p, {np.float64: 0, np.float32: 1}[dt] if prec is None else 2).kernel, f"{err:.2e}")
        ok &= err < 5e-3
for (m, n, p) in [(1920, 1024, 1920), (2000, 48, 2000), (7040, 16, 7040)]:
    A = I.host_matrix(m, n, 3, I.ID_A); B = I.host_matrix(n, p, 3, I.ID_B)
    C = moa.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    same = bool(np.all(C == O.ip(A, B, fused=True)))
    pl = moa.plan(m, n, p)
    print(m, n, p, "float64 K1", pl.bm, pl.bn, "tiles", pl.tiles, "grid", pl.grid, "bitwise" if same else "MISMATCH")
    ok &= same
# latency tiles: one-shot (n <= 256: 256^3 and 200x96x260 above) in accumulate mode as a
# two-panel chain, and the ring-fed latency tile (n > 256)
for (m, n, p, k0) in [(200, 96, 260, 48), (300, 512, 300, 0)]:
    A = I.host_matrix(m, n, 5, I.ID_A); B = I.host_matrix(n, p, 5, I.ID_B)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.zeros((m, p), dtype=torch.float64, device="cuda")
    if k0:
        moa.gemm_acc(Ad[:, :k0], Bd[:k0], C, True)
        moa.gemm_acc(Ad[:, k0:], Bd[k0:], C, True)
    else:
        C = moa.gemm(Ad, Bd)
    torch.cuda.synchronize()
    pl = moa.plan(m, n, p)
    same = bool(np.all(C.cpu().numpy() == O.ip(A, B, fused=True)))
    print(m, n, p, "float64 latency tile", pl.bm, pl.bn, pl.stages, "acc chain" if k0 else "", "bitwise" if same else "MISMATCH")
    ok &= same
# fused-gather epilogue (K1/K2 PEER): 3 extra destinations, stream-K and generic shapes
for (m, n, p) in [(2000, 48, 2000), (130, 34, 66), (257, 33, 131)]:
    A = I.host_matrix(m, n, 4, I.ID_A); B = I.host_matrix(n, p, 4, I.ID_B)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.empty((m, p), dtype=torch.float64, device="cuda")
    dst = [torch.empty((m, p), dtype=torch.float64, device="cuda") for _ in range(3)]
    moa.gemm_scatter(Ad, Bd, C, dst)
    torch.cuda.synchronize()
    ref = O.ip(A, B, fused=True)
    same = bool(np.all(C.cpu().numpy() == ref)) and all(bool(torch.equal(d, C)) for d in dst)
    print(m, n, p, "float64 scatter x3", "bitwise" if same else "MISMATCH")
    ok &= same
# K3 / K3g with the same epilogue (fp32 exact)
for (m, n, p) in [(300, 96, 260), (129, 33, 131)]:
    A = I.host_matrix(m, n, 4, I.ID_A, dtype=np.float32); B = I.host_matrix(n, p, 4, I.ID_B, dtype=np.float32)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.empty((m, p), dtype=torch.float32, device="cuda")
    dst = [torch.empty((m, p), dtype=torch.float32, device="cuda") for _ in range(2)]
    moa.gemm_scatter(Ad, Bd, C, dst)
    torch.cuda.synchronize()
    same = bool(np.all(C.cpu().numpy() == O.ip(A, B, fused=True))) and all(bool(torch.equal(d, C)) for d in dst)
    print(m, n, p, "float32 scatter x2", "bitwise" if same else "MISMATCH")
    ok &= same
print("ALL OK" if ok else "MISMATCH")
