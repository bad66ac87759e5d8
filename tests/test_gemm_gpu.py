"""GPU parity of the fp64 MoA-ONF GEMM (C ABI via the binding) against the CPU oracle.

Bars (north_star + DESIGN.md §Parity):
  * bitwise vs oracle ``ip(fused=True)`` (Fig. 3 ip.c with the update fused,
    reading R3) on ANY finite input — the kernels keep k strictly ascending and
    DMMA.8x8x4 is an fma chain (profiles/r01_fp64_probe.jsonl);
  * bitwise vs the unfused literal ip.c on integer-valued inputs;
  * relative Frobenius error vs the unfused literal ip.c <= 1e-12 * sqrt(n).
Large shapes (the bench configs) are checked on sampled rows (rows of C are
independent, Fig. 1 / P:99) plus a Freivalds product check.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from inputs import inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu

EDGE = [1, 2, 3, 7, 8, 9, 15, 16, 17, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257]
# every compiled K1 tile config (bm, bn, stages), incl. the latency tiles
K1_CONFIGS = [(128, 128, 6), (128, 64, 4), (64, 64, 4), (64, 32, 4), (16, 32, 4), (16, 16, 4),
              # latency tiles with 8x16 warp tiles (stages 8 tells them apart)
              (16, 32, 8), (16, 16, 8),
              # their one-shot twins (16 stages: all of k <= 256 resident)
              (16, 32, 16), (16, 16, 16)]


def _moa():
    import paper_2306_11148_b200 as moa
    return moa


def _host(m, n, p, seed, kind=I.UNIFORM, dtype=np.float64):
    A = I.host_matrix(m, n, seed, I.ID_A, kind, dtype)
    B = I.host_matrix(n, p, seed, I.ID_B, kind, dtype)
    return A, B


def _gpu_gemm(A, B, dev, precision=None):
    import torch
    tA = torch.from_numpy(A).to(dev)
    tB = torch.from_numpy(B).to(dev)
    C = _moa().gemm(tA, tB, precision=precision)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def _bits_equal(x, y):
    # == semantics (±0 equal), and no NaNs expected
    return x.shape == y.shape and bool(np.all(x == y))


def _relfro(x, ref):
    d = np.linalg.norm((x - ref).ravel())
    r = np.linalg.norm(ref.ravel())
    return d / r if r > 0 else d


def test_config0_square_256_vs_oracle(cuda_device):
    """BASELINE configs[0]: m=n=p=256 fp64 against the full oracle, seeds 1-3."""
    for seed in (1, 2, 3):
        A, B = _host(256, 256, 256, seed)
        C = _gpu_gemm(A, B, cuda_device)
        assert _bits_equal(C, O.ip(A, B, fused=True)), seed
        assert _relfro(C, O.ip(A, B, fused=False)) <= 1e-12 * np.sqrt(256)
        Ai, Bi = _host(256, 256, 256, seed, kind=I.INT)
        assert _bits_equal(_gpu_gemm(Ai, Bi, cuda_device), O.ip(Ai, Bi, fused=False))


@pytest.mark.parametrize("seed", [1, 2])
def test_tile_edge_shapes(cuda_device, seed):
    """Shapes straddling every tile/box/atom edge, even (TMA kernel) and odd (generic kernel)."""
    rng = np.random.default_rng(100 + seed)
    shapes = {(m, n, p) for m in (1, 129, 257) for n in (1, 17, 64) for p in (2, 130, 256)}
    shapes |= {tuple(int(x) for x in rng.choice(EDGE, size=3)) for _ in range(30)}
    for (m, n, p) in sorted(shapes):
        A, B = _host(m, n, p, seed)
        C = _gpu_gemm(A, B, cuda_device)
        assert _bits_equal(C, O.ip(A, B, fused=True)), (m, n, p)
        assert _relfro(C, O.ip(A, B, fused=False)) <= 1e-12 * np.sqrt(n), (m, n, p)


def test_generic_kernel_on_misaligned_pointers(cuda_device):
    """Element-aligned but not 16-byte aligned operands route to the generic kernel:
    same bits."""
    import torch
    moa = _moa()
    m, n, p = 70, 46, 38
    A, B = _host(m, n, p, 4)
    bufA = torch.empty(m * n + 1, dtype=torch.float64, device=cuda_device)
    bufB = torch.empty(n * p + 1, dtype=torch.float64, device=cuda_device)
    bufC = torch.empty(m * p + 1, dtype=torch.float64, device=cuda_device)
    tA = bufA[1:].view(m, n)
    tB = bufB[1:].view(n, p)
    tC = bufC[1:].view(m, p)
    tA.copy_(torch.from_numpy(A))
    tB.copy_(torch.from_numpy(B))
    moa.gemm(tA, tB, out=tC)
    torch.cuda.synchronize()
    assert _bits_equal(tC.cpu().numpy(), O.ip(A, B, fused=True))


def test_identities_bitwise(cuda_device):
    m, n, p = 200, 96, 130
    A, B = _host(m, n, p, 5)
    assert _bits_equal(_gpu_gemm(A, np.eye(n), cuda_device), A)
    assert _bits_equal(_gpu_gemm(np.eye(m), A, cuda_device), A)
    assert _bits_equal(_gpu_gemm(A, np.zeros((n, p)), cuda_device), np.zeros((m, p)))
    C = _gpu_gemm(A, B, cuda_device)
    Ct = _gpu_gemm(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T), cuda_device)
    assert _bits_equal(C.T, Ct)  # products commute exactly, same k order


def test_rank1_closed_form(cuda_device):
    rng = np.random.default_rng(6)
    m, n, p = 300, 250, 170
    u, z = rng.integers(-2, 3, size=m), rng.integers(-2, 3, size=p)
    v, w = rng.integers(-1, 2, size=n), rng.integers(-1, 2, size=n)
    A, B = np.outer(u, v).astype(np.float64), np.outer(w, z).astype(np.float64)
    C = _gpu_gemm(A, B, cuda_device)
    assert _bits_equal(C, np.outer(u, z).astype(np.float64) * float(v @ w))


def test_zero_extents(cuda_device):
    import torch
    moa = _moa()
    A = torch.empty((5, 0), dtype=torch.float64, device=cuda_device)
    B = torch.empty((0, 7), dtype=torch.float64, device=cuda_device)
    C = torch.full((5, 7), 3.0, dtype=torch.float64, device=cuda_device)
    moa.gemm(A, B, out=C)
    torch.cuda.synchronize()
    assert torch.all(C == 0)
    A0 = torch.empty((0, 4), dtype=torch.float64, device=cuda_device)
    B0 = torch.ones((4, 3), dtype=torch.float64, device=cuda_device)
    assert moa.gemm(A0, B0).shape == (0, 3)


def test_aliasing_rejected(cuda_device):
    import torch
    moa = _moa()
    A = torch.ones((64, 64), dtype=torch.float64, device=cuda_device)
    B = torch.ones((64, 64), dtype=torch.float64, device=cuda_device)
    with pytest.raises(moa.MoAError) as e:
        moa.gemm(A, B, out=A)
    assert e.value.name == "MOA_ERR_ALIASING"


def test_row_block_invariance_and_determinism(cuda_device):
    """F8: any row block computed alone is bitwise the same rows of the full product,
    and two runs are bitwise equal (no atomics, k order fixed by n alone)."""
    import torch
    moa = _moa()
    m, n, p = 1000, 520, 384
    A, B = _host(m, n, p, 7)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    full = moa.gemm(tA, tB)
    again = moa.gemm(tA, tB)
    torch.cuda.synchronize()
    assert torch.equal(full, again)
    for (r0, r1) in [(0, 1), (0, 500), (333, 1000), (999, 1000), (128, 256), (7, 700)]:
        part = moa.gemm(tA[r0:r1].contiguous(), tB)
        torch.cuda.synchronize()
        assert torch.equal(part, full[r0:r1]), (r0, r1)


def test_each_compiled_tile_config_bitwise(cuda_device):
    """The block-size sweep configs (the paper's block-size experiment) all compute the
    same bits — the plan changes only the lifting, never the k order."""
    import torch
    moa = _moa()
    m, n, p = 300, 200, 260
    A, B = _host(m, n, p, 8)
    ref = O.ip(A, B, fused=True)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    base = moa.plan(m, n, p)
    assert base.kernel == "dgemm_tma"
    for (bm, bn, st) in K1_CONFIGS:
        pl = moa.Plan(**{**base.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
        out = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
        moa.gemm_with_plan(tA, tB, out, pl)
        torch.cuda.synchronize()
        assert _bits_equal(out.cpu().numpy(), ref), (bm, bn, st)


@pytest.mark.parametrize("shape", [(256, 256, 256), (250, 256, 250), (1, 16, 2), (17, 254, 34), (160, 48, 480),
                                   (300, 200, 260), (512, 512, 512), (96, 600, 130), (384, 64, 384)])
def test_latency_tiles_bitwise(cuda_device, shape):
    """Tiny problems (configs[0], 256^3): the chooser's latency tiles (16x16 of two 8x16
    warps up to 2.75 tiles per SM, then 16x32 of four 8x16 warps up to 2 per SM, then
    16x32 of two 16x16 warps; one tile per CTA; for n <= 256 the one-shot twins with all
    of k resident, whichever streams fewer bytes into the busiest SM) give the fused ip.c bits, ragged edges
    included, and the literal ip.c within 1e-12 sqrt(n); every latency config does;
    a two-panel accumulate chain started from +0 is the same chain; the fused-gather
    epilogue writes the same bits to an extra destination."""
    import torch
    moa = _moa()
    m, n, p = shape
    A, B = _host(m, n, p, 31)
    ref = O.ip(A, B, fused=True)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    pl = moa.plan(m, n, p)
    t16, t32 = -(-m // 16) * -(-p // 16), -(-m // 16) * -(-p // 32)
    want = (16, 16, 8) if 4 * t16 <= 11 * pl.sms else ((16, 32, 8) if t32 <= 2 * pl.sms else (16, 32, 4))
    if want[2] == 8 and -(-n // 16) <= 16:  # one-shot twins: all of k resident, one tile per CTA
        ok16, ok32 = t16 <= 3 * pl.sms, t32 <= 2 * pl.sms  # 64 / 96 KiB of smem per CTA
        b16, b32 = -(-t16 // pl.sms) * 32, -(-t32 // pl.sms) * 48
        if ok32 and (not ok16 or b32 < b16):
            want = (16, 32, 16)
        elif ok16:
            want = (16, 16, 16)
    assert (pl.bm, pl.bn, pl.stages) == want, pl
    assert pl.grid == pl.tiles
    got = moa.gemm(tA, tB).cpu().numpy()
    assert _bits_equal(got, ref)
    lit = O.ip(A, B, fused=False)
    assert np.linalg.norm(got - lit) <= 1e-12 * np.sqrt(n) * np.linalg.norm(lit)
    for (bm, bn, st) in [c for c in K1_CONFIGS if c[0] == 16]:
        q = moa.Plan(**{**pl.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
        out = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
        moa.gemm_with_plan(tA, tB, out, q)
        torch.cuda.synchronize()
        assert _bits_equal(out.cpu().numpy(), ref), (bm, bn)
    k0 = (n // 2) // 2 * 2
    out = torch.zeros((m, p), dtype=torch.float64, device=cuda_device)
    moa.gemm_acc(tA[:, :k0], tB[:k0], out, True)
    moa.gemm_acc(tA[:, k0:], tB[k0:], out, True)
    torch.cuda.synchronize()
    assert _bits_equal(out.cpu().numpy(), ref)
    D = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
    Cd = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
    moa.gemm_scatter(tA, tB, Cd, [D])
    torch.cuda.synchronize()
    assert _bits_equal(Cd.cpu().numpy(), ref) and _bits_equal(D.cpu().numpy(), ref)
    # the accumulate + extra-destination instantiation (the last k-panel of a gathered
    # chain), on the same latency / one-shot tiles
    D2 = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
    C2 = torch.zeros((m, p), dtype=torch.float64, device=cuda_device)
    moa.gemm_acc(tA[:, :k0], tB[:k0], C2, True)
    moa.gemm_scatter(tA[:, k0:], tB[k0:], C2, [D2], accumulate=True)
    torch.cuda.synchronize()
    assert _bits_equal(C2.cpu().numpy(), ref) and _bits_equal(D2.cpu().numpy(), ref)


@pytest.mark.parametrize("shape", [(2000, 200, 2000), (1500, 100, 3000), (2100, 56, 1030)])
def test_stream_k_split_tiles_bitwise(cuda_device, shape):
    """Stream-K (moa_ptx.cuh sk_plan): tiles cut along k between two CTAs, the high-k
    part continuing the chain from the stored low-k partial, are bitwise the fused
    ip.c result — for every compiled tile config, with ragged k (n % 16 != 0), and in
    accumulate mode (C := C0 + A.B, chain started from C0)."""
    import torch
    moa = _moa()
    m, n, p = shape
    A, B = _host(m, n, p, 21)
    ref = O.ip(A, B, fused=True)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    base = moa.plan(m, n, p)
    split_seen = False
    for (bm, bn, st) in K1_CONFIGS:
        pl = moa.Plan(**{**base.__dict__, "bm": bm, "bn": bn, "stages": st, "grid": 0})
        out = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
        moa.gemm_with_plan(tA, tB, out, pl)
        torch.cuda.synchronize()
        assert _bits_equal(out.cpu().numpy(), ref), (bm, bn, st)
        tiles = -(-m // bm) * -(-p // bn)
        split_seen |= tiles >= pl.sms and tiles % pl.sms != 0
    assert split_seen
    # accumulate mode: two k-panels through moa_gemm_acc equal the one-call chain
    k1 = 48
    C = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
    moa.gemm_acc(tA[:, :k1], tB[:k1], C, accumulate=False)
    moa.gemm_acc(tA[:, k1:], tB[k1:], C, accumulate=True)
    torch.cuda.synchronize()
    assert _bits_equal(C.cpu().numpy(), ref)


def test_plan_is_static_and_sane(cuda_device):
    moa = _moa()
    for (m, n, p) in [(256, 256, 256), (1024, 1024, 1024), (8192, 8192, 8192), (16384, 16384, 16384),
                      (65536, 512, 512)]:
        pl = moa.plan(m, n, p)
        assert pl.kernel == "dgemm_tma" and pl.bk == 16, pl
        assert pl.tiles == -(-m // pl.bm) * -(-p // pl.bn)
        assert 1 <= pl.grid <= max(pl.tiles, pl.sms * pl.ctas_per_sm) and pl.ctas_per_sm >= 1
        assert moa.plan(m, n, p) == pl
    assert moa.plan(16384, 16384, 16384).bm == 128
    # measured picks (profiles/r02/ab_midn_grid.jsonl, small_n_oneshot.json): one wave of
    # 128x64 tiles at N = 1024; the one-shot 16x32 latency tile at configs[0]
    q = moa.plan(1024, 1024, 1024)
    assert (q.bm, q.bn) == (128, 64), q
    q = moa.plan(256, 256, 256)
    assert (q.bm, q.bn, q.stages) == (16, 32, 16), q
    assert moa.plan(5, 7, 9).kernel == "dgemm_generic"  # odd n / p: not describable by TMA
    # thin p (the HBM-bound diagnostic m = 2^20, n = p = 32): a 32-column tile, no
    # wasted DMMA columns; near-square shapes keep the wide tiles
    for (m, n, p) in [(1 << 20, 32, 32), (1 << 20, 16, 16), (1 << 18, 128, 32), (1 << 20, 96, 96)]:
        assert moa.plan(m, n, p).bn == 32, (m, n, p)
    for (m, n, p) in [(8224, 8224, 8224), (1 << 20, 64, 64), (4096, 4096, 4096)]:
        assert moa.plan(m, n, p).bn >= 64, (m, n, p)


def _freivalds(Ct, tA, tB, trials=2):
    """y = C x vs z = A (B x) on the GPU in fp64 with x in {+-1}^p: O(N^2) check of every element."""
    import torch
    worst = 0.0
    for t in range(trials):
        g = torch.Generator(device="cpu").manual_seed(1234 + t)
        x = (torch.randint(0, 2, (Ct.shape[1], 1), generator=g) * 2 - 1).to(Ct)
        y = Ct @ x
        z = tA @ (tB @ x)
        worst = max(worst, float(torch.linalg.norm(y - z) / torch.linalg.norm(z)))
    return worst


@pytest.mark.parametrize("cfg", ["square8192", "skinny65536x512"])
def test_bench_configs_sampled_rows(cuda_device, cfg):
    """At the full BASELINE sizes in the launch configuration bench.py times: sampled rows
    bitwise vs the oracle (tile-boundary rows included) + Freivalds on the whole of C."""
    import torch
    moa = _moa()
    m, n, p = (8192, 8192, 8192) if cfg == "square8192" else (65536, 512, 512)
    seed = 1
    tA = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
    tB = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
    I.device_fill(tA, seed, I.ID_A)
    I.device_fill(tB, seed, I.ID_B)
    C = moa.gemm(tA, tB)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    rows = sorted({0, m - 1, 127, 128, 129, m // 2, m // 2 + 1, *rng.integers(0, m, size=9).tolist()})
    B = I.host_matrix(n, p, seed, I.ID_B)
    Arows = I.host_rows(rows, n, seed, I.ID_A)
    ref = O.ip_rowblock(Arows, B, fused=True)
    got = C[torch.tensor(rows, device=cuda_device)].cpu().numpy()
    assert _bits_equal(got, ref)
    assert _freivalds(C, tA, tB) <= 1e-12 * np.sqrt(n)


@pytest.mark.parametrize("shape", [(333, 128, 210), (4000, 256, 2048)])
def test_gemm_host_e2e(cuda_device, shape):
    """moa_gemm_host (row-panel pipelined H2D / compute / D2H): same bits as the oracle."""
    import torch
    moa = _moa()
    m, n, p = shape
    A, B = _host(m, n, p, 9)
    hA = torch.from_numpy(A).pin_memory()
    hB = torch.from_numpy(B).pin_memory()
    hC = torch.empty((m, p), dtype=torch.float64).pin_memory()
    dA = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
    dB = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
    dC = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
    moa.gemm_host(hA, hB, hC, dA, dB, dC)
    assert _bits_equal(hC.numpy(), O.ip(A, B, fused=True))


@pytest.mark.parametrize("shape", [(6400, 1024, 256), (6144, 24576, 64)])
def test_gemm_host_e2e_chained_first_panel(cuda_device, shape):
    """moa_gemm_host when row panel 0 is chained over B's k-panels while B crosses the
    host link (m >= 2 x ~2.9K rows, n >= 512: 8 panels; n >= 24576: 16): the same bits
    as the one-call device GEMM, and sampled rows as the oracle."""
    import torch
    moa = _moa()
    m, n, p = shape
    dA = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
    dB = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
    I.device_fill(dA, 13, I.ID_A)
    I.device_fill(dB, 13, I.ID_B)
    ref = moa.gemm(dA, dB).cpu()
    hA, hB = dA.cpu().pin_memory(), dB.cpu().pin_memory()
    hC = torch.full((m, p), float("nan"), dtype=torch.float64).pin_memory()
    dA2 = torch.full_like(dA, float("nan"))
    dB2 = torch.full_like(dB, float("nan"))
    dC2 = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
    moa.gemm_host(hA, hB, hC, dA2, dB2, dC2)
    assert torch.equal(hC, ref)
    rows = [0, 1, 2943, 2944, 2945, m // 2, m - 1]
    got = hC.numpy()[rows]
    assert _bits_equal(got, O.ip_rowblock(hA.numpy()[rows], hB.numpy(), fused=True))


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_k_panel_chain_is_bitwise_one_launch(cuda_device, dtype):
    """moa_gemm_acc: C := A[:, :k1] • B[:k1]; C += A[:, k1:] • B[k1:] ... reproduces the
    one-launch C bit for bit — the blocked sigma loop with its 'addition loop'
     across launches. Split points include ones that break 16-byte
    alignment (generic kernel for that panel): same arithmetic, same bits."""
    import torch
    moa = _moa()
    tdt = torch.float64 if dtype == "f64" else torch.float32
    ndt = np.float64 if dtype == "f64" else np.float32
    m, n, p = 300, 520, 264
    A = I.host_matrix(m, n, 21, I.ID_A, dtype=ndt)
    B = I.host_matrix(n, p, 21, I.ID_B, dtype=ndt)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    full = moa.gemm(tA, tB)
    for cuts in ([0, 256, 520], [0, 32, 64, 320, 520], [0, 37, 300, 301, 520], [0, 520]):
        C = torch.full((m, p), float("nan"), dtype=tdt, device=cuda_device)
        for j in range(len(cuts) - 1):
            k0, k1 = cuts[j], cuts[j + 1]
            moa.gemm_acc(tA[:, k0:k1], tB[k0:k1], C, accumulate=j > 0)
        torch.cuda.synchronize()
        assert torch.equal(C, full), cuts
    ref = O.ip(A, B, fused=True)
    assert np.array_equal(full.cpu().numpy(), ref)


def test_strided_output_and_validation(cuda_device):
    import torch
    moa = _moa()
    m, n, p = 130, 64, 96
    A, B = _host(m, n, p, 22)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    big = torch.full((m, p + 10), -1.0, dtype=torch.float64, device=cuda_device)
    moa.gemm_acc(tA, tB, big[:, 2:2 + p], accumulate=False)
    torch.cuda.synchronize()
    assert _bits_equal(big[:, 2:2 + p].cpu().numpy(), O.ip(A, B, fused=True))
    assert torch.all(big[:, :2] == -1) and torch.all(big[:, 2 + p:] == -1)
    rc = moa._moa_gemm_acc(m, n, p, tA.data_ptr(), n - 1, tB.data_ptr(), p, big.data_ptr(), p + 10, 0, 0, None)
    assert rc == 1  # lda < n


@pytest.mark.gpu
def test_pure_c_caller_through_the_abi(cuda_device, tmp_path):
    """The boundary without Python or torch: a C99 program allocates with the CUDA
    runtime, calls moa_gemm on integer-valued fp64 data (every summation order gives
    the same bits, pin P6) and compares with its own triple loop exactly."""
    import shutil
    import subprocess
    import paper_2306_11148_b200 as moa
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    src = tmp_path / "c_gemm.c"
    src.write_text(r"""
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include "moa.h"
int main(void) {
  const int64_t m = 300, n = 200, p = 260;
  double *hA = malloc(sizeof(double) * m * n), *hB = malloc(sizeof(double) * n * p);
  double *hC = malloc(sizeof(double) * m * p), *dA, *dB, *dC;
  for (int64_t i = 0; i < m * n; ++i) hA[i] = (double)((i * 7 + 3) % 9) - 4.0;
  for (int64_t i = 0; i < n * p; ++i) hB[i] = (double)((i * 5 + 1) % 9) - 4.0;
  if (cudaMalloc((void**)&dA, sizeof(double) * m * n) || cudaMalloc((void**)&dB, sizeof(double) * n * p) ||
      cudaMalloc((void**)&dC, sizeof(double) * m * p)) return 10;
  cudaMemcpy(dA, hA, sizeof(double) * m * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(double) * n * p, cudaMemcpyHostToDevice);
  int rc = moa_gemm(m, n, p, dA, dB, dC, MOA_F64, NULL);
  if (rc != MOA_OK) { printf("moa_gemm: %s %s\n", moa_status_string(rc), moa_last_error()); return 11; }
  if (cudaDeviceSynchronize() != cudaSuccess) return 12;
  cudaMemcpy(hC, dC, sizeof(double) * m * p, cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < p; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s += hA[i * n + k] * hB[k * p + j];
      if (s != hC[i * p + j]) { printf("mismatch at %ld %ld\n", (long)i, (long)j); return 13; }
    }
  printf("C GEMM OK\n");
  return 0;
}
""")
    libdir = os.path.dirname(moa.lib_path)
    exe = tmp_path / "c_gemm"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                        str(src), "-o", str(exe), "-L", libdir, "-l:libmoa.so", "-L", "/usr/local/cuda/lib64",
                        "-lcudart", "-Wl,-rpath," + libdir + ":/usr/local/cuda/lib64"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "C GEMM OK" in r.stdout, (r.returncode, r.stdout, r.stderr)
