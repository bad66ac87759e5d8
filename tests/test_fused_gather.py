"""Row-lifted GEMM with the all-gather of C fused into the GEMM epilogue (SURVEY
§8(f) NEXT-1 step 3; reading R14): moa_gemm_scatter (the epilogue on one GPU),
the symmetric-window helpers and moa_gemm_lifted_gather.

Rows of C depend only on the same rows of A and on all of B (Fig. 1), so the
gathered C_full equals the one-GPU product; every destination of the epilogue must
hold exactly the oracle's bits (fused ip.c, reading R3).

CPU (`-m "not gpu"`): argument validation happens before any CUDA call.
GPU: the scatter epilogue with up to 8 destinations on every schedule (latency
tiles, 128x128 dynamic + stream-K with split tiles, the generic kernel, n = 0,
accumulate chains), and the full collective path on a 1-rank NCCL communicator
(window allocation, peer-address resolution, barriers, lifted compute).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2306_11148_b200 as moa
from inputs import inputs as I
from oracle import oracle as O


def test_scatter_validation_without_gpu():
    A, B, C, D = 0x10000, 0x200000, 0x4000000, 0x8000000
    arr = (moa._vp * 9)(*([D + i * 0x100000 for i in range(9)]))
    f = moa._moa_gemm_scatter
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 9, arr, 0, None) == 1            # ndst > 8
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, -1, arr, 0, None) == 1           # ndst < 0
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 1, arr, 3, None) == 2            # unknown dtype
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 1, None, 0, None) == 3           # NULL dst array
    bad = (moa._vp * 2)(D, None)
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 2, bad, 0, None) == 3            # NULL destination
    mis = (moa._vp * 1)(D + 4)
    assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 1, mis, 0, None) == 5            # misaligned
    for q in (C + 8, A + 16, B, D):
        al = (moa._vp * 2)(D, q)
        assert f(4, 8, 8, A, 8, B, 8, C, 8, 0, 2, al, 0, None) == 4         # overlaps C / A / B / dst[0]
    assert f(4, 8, 8, A, 7, B, 8, C, 8, 0, 1, arr, 0, None) == 1            # lda < n (as moa_gemm_acc)
    # the collective entry points: NULL communicator before anything else
    assert moa._moa_gemm_lifted_gather(4, 4, 4, A, B, C, 0, None, None, 0) == 3
    assert moa._moa_comm_alloc_window(None, 64, moa._vp()) == 3
    assert moa._moa_status_string(10) == b"MOA_ERR_NOT_REGISTERED"
    assert moa._moa_gemm_lifted_2d_gather(4, 4, 4, 1, 1, A, B, C, D, 0, None, None) == 3
    assert moa._moa_gemm_lifted_host(4, 4, 4, A, B, C, A, B, C, 0, None, None) == 3
    assert moa._moa_comm_window_peer(None, A, 0, moa._vp()) == 3
    assert moa._moa_comm_free_window(None, A) == 3


# --------------------------------------------------------------------- GPU ----

def _operands(m, n, p, seed, dev):
    A = torch.empty((m, n), dtype=torch.float64, device=dev)
    B = torch.empty((n, p), dtype=torch.float64, device=dev)
    if m * n:
        I.device_fill(A, seed, I.ID_A)
    if n * p:
        I.device_fill(B, seed, I.ID_B)
    return A, B


# (shape, what it exercises, the chooser's (bm, bn) for it or None)
_SHAPES = [
    ((200, 144, 176), "latency tiles 16x16", (16, 16)),
    ((512, 96, 512), "latency tiles 16x32", (16, 32)),
    ((1920, 1024, 1920), "128x128 stream-K only (split tiles)", (128, 128)),
    ((2560, 1024, 2560), "128x128 dynamic tiles + stream-K runs", (128, 128)),
    ((2000, 48, 2000), "64x32 shallow k, stream-K over 3 CTAs per SM", (64, 32)),
    ((1000, 256, 300), "ragged tail", None),
    ((257, 33, 131), "generic kernel (odd n, p)", None),
    ((300, 0, 200), "n = 0: zero fill", None),
]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,what,tile", _SHAPES, ids=[w for _, w, _ in _SHAPES])
def test_scatter_every_destination_bitwise(cuda_device, shape, what, tile):
    m, n, p = shape
    if tile is not None:  # the schedule this case is meant to exercise
        pl = moa.plan(m, n, p)
        assert (pl.bm, pl.bn) == tile, (what, pl)
    A, B = _operands(m, n, p, 7, cuda_device)
    ref = O.ip(A.cpu().numpy(), B.cpu().numpy(), fused=True) if n else np.zeros((m, p))
    for nd in (1, 3, 8):
        C = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
        dst = [torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device) for _ in range(nd)]
        moa.gemm_scatter(A, B, C, dst)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), ref), (what, nd)
        for d, t in enumerate(dst):
            assert torch.equal(t, C), (what, nd, d)
    # ndst = 0 is plain moa_gemm (the non-PEER kernel)
    C0 = moa.gemm_scatter(A, B, torch.empty((m, p), dtype=torch.float64, device=cuda_device), [])
    torch.cuda.synchronize()
    assert np.array_equal(C0.cpu().numpy(), ref)


@pytest.mark.gpu
def test_scatter_accumulate_chain_last_panel(cuda_device):
    """The lifted path's pipelined k-panels: panel j > 0 continues every element's fma
    chain from C; only the last panel (accumulate + destinations, K1 ACC+PEER) writes
    the destinations, which must hold the one-launch bits."""
    for (m, n, p) in [(1000, 1000, 300), (2000, 96, 2000), (129, 70, 131)]:
        A, B = _operands(m, n, p, 8, cuda_device)
        ref = moa.gemm(A, B)
        C = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
        dst = [torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device) for _ in range(2)]
        cuts = [0, (n // 3) // 32 * 32, (2 * n // 3) // 32 * 32, n]
        for j in range(3):
            k0, k1 = cuts[j], cuts[j + 1]
            moa.gemm_scatter(A[:, k0:k1], B[k0:k1, :], C, dst if j == 2 else [], accumulate=j > 0)
        torch.cuda.synchronize()
        assert torch.equal(C, ref), (m, n, p)
        for t in dst:
            assert torch.equal(t, ref), (m, n, p)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(2000, 64, 2048), (300, 200, 260), (257, 33, 131)],
                         ids=["k3-multiwave", "k3-ragged", "k3-generic"])
def test_scatter_fp32_exact_bitwise(cuda_device, shape):
    """K3 / K3g PEER epilogue: fp32 exact (fused fma chain, k ascending) in every
    destination, bitwise the fp32 fused oracle."""
    m, n, p = shape
    A = torch.from_numpy(I.host_matrix(m, n, 3, I.ID_A, dtype=np.float32)).to(cuda_device)
    B = torch.from_numpy(I.host_matrix(n, p, 3, I.ID_B, dtype=np.float32)).to(cuda_device)
    ref = O.ip(A.cpu().numpy(), B.cpu().numpy(), fused=True)
    C = torch.full((m, p), float("nan"), dtype=torch.float32, device=cuda_device)
    dst = [torch.full((m, p), float("nan"), dtype=torch.float32, device=cuda_device) for _ in range(3)]
    moa.gemm_scatter(A, B, C, dst)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), ref)
    for t in dst:
        assert torch.equal(t, C)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(512, 256, 384), (300, 200, 260), (129, 33, 131)])
def test_scatter_3xtf32(cuda_device, shape):
    """The 3xTF32 tcgen05 kernel (K4) carries the fused-gather epilogue too: every
    destination holds exactly the bits of C, C is within the variant's tolerance of the
    literal oracle (5e-3, north_star) and at fp32 level vs the fp64 truth; a two-panel
    accumulate chain scatters its final sums. (129x33x131 is not TMA-describable: the
    exact fp32 generic kernel takes it, reading R20.)"""
    m, n, p = shape
    A = I.host_matrix(m, n, 7, I.ID_A, I.UNIFORM, np.float32)
    B = I.host_matrix(n, p, 7, I.ID_B, I.UNIFORM, np.float32)
    tA, tB = torch.from_numpy(A).to(cuda_device), torch.from_numpy(B).to(cuda_device)
    if (m, n, p) != (129, 33, 131):
        assert moa.plan(m, n, p, moa.F32_3XTF32).kernel == "sgemm_3xtf32"
    C = torch.empty((m, p), dtype=torch.float32, device=cuda_device)
    dst = [torch.full((m, p), float("nan"), dtype=torch.float32, device=cuda_device) for _ in range(3)]
    moa.gemm_scatter(tA, tB, C, dst, precision="3xtf32")
    torch.cuda.synchronize()
    for t in dst:
        assert torch.equal(t, C)
    lit = O.ip(A, B, fused=False)
    got = C.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(got - lit) <= 5e-3 * np.linalg.norm(lit)
    truth = O.ip_f32_truth(A, B)
    assert np.linalg.norm(got - truth) <= 1e-5 * np.sqrt(n) * np.linalg.norm(truth)
    k0 = (n // 2) // 8 * 8 or n
    C2 = torch.zeros((m, p), dtype=torch.float32, device=cuda_device)
    d2 = torch.full((m, p), float("nan"), dtype=torch.float32, device=cuda_device)
    moa.gemm_acc(tA[:, :k0], tB[:k0], C2, True, precision="3xtf32")
    if k0 < n:
        moa.gemm_scatter(tA[:, k0:], tB[k0:], C2, [d2], accumulate=True, precision="3xtf32")
    else:
        moa.gemm_scatter(tA[:, :0], tB[:0], C2, [d2], accumulate=True, precision="3xtf32")
    torch.cuda.synchronize()
    assert torch.equal(d2, C2)
    assert np.linalg.norm(C2.cpu().numpy().astype(np.float64) - truth) <= 1e-5 * np.sqrt(n) * np.linalg.norm(truth)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.gpu
def test_lifted_gather_single_rank_nccl(cuda_device):
    """The whole collective path on a 1-rank NCCL communicator: symmetric window
    allocation and peer-address resolution (rank 0's own copy resolves to the local
    pointer), entry/exit barriers, B broadcast (pipelined panels too) and the lifted
    compute into C_full — bitwise moa_gemm."""
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        for (m, n, p) in [(1000, 256, 300), (2000, 48, 2000), (129, 64, 130)]:
            A, B = _operands(m, n, p, 9, cuda_device)
            ref = moa.gemm(A, B)
            C_full = comm.alloc_window((m, p))
            # rank 0's resolved address (NCCL's flat LSA mapping) aliases the same memory:
            # the epilogue storing through it lands in C_full
            peer0 = comm.window_peer(C_full, 0)
            assert comm.window_peer(C_full[1:], 0) == peer0 + p * 8
            C_full.fill_(float("nan"))
            C_tmp = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
            moa.gemm_scatter(A, B, C_tmp, [peer0])
            torch.cuda.synchronize()
            assert torch.equal(C_full, ref) and torch.equal(C_tmp, ref)
            for K in (0, 3):
                C_full.fill_(float("nan"))
                moa.gemm_lifted_gather(m, A, B, C_full, comm, npanels=K)
                torch.cuda.synchronize()
                assert torch.equal(C_full, ref), (m, n, p, K)
            comm.free_window(C_full)
        # C_full outside any window
        A, B = _operands(64, 32, 64, 1, cuda_device)
        plain = torch.empty((64, 64), dtype=torch.float64, device=cuda_device)
        with pytest.raises(moa.MoAError) as e:
            moa.gemm_lifted_gather(64, A, B, plain, comm)
        assert e.value.name == "MOA_ERR_NOT_REGISTERED"
        # fp32 exact through the same collective path (K3 PEER)
        w = comm.alloc_window((64, 64), torch.float32)
        w.fill_(float("nan"))
        moa.gemm_lifted_gather(64, A.float(), B.float(), w, comm)
        torch.cuda.synchronize()
        assert torch.equal(w, moa.gemm(A.float(), B.float()))
        with pytest.raises(moa.MoAError) as e:
            comm.window_peer(plain, 0)
        assert e.value.name == "MOA_ERR_NOT_REGISTERED"
    finally:
        comm.close()
        dist.destroy_process_group()


def _ipc_worker(rank, world, m, n, p, q_out, q_in, barrier, result):
    """One 'rank' of a two-process gather on one GPU: its C_full travels to the other
    process by CUDA IPC, and each process's epilogue stores its rows into both copies
    (the address arithmetic of moa_gemm_lifted_gather, with IPC standing in for the
    NCCL window's NVLink mapping)."""
    import torch
    import numpy as np
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    from oracle import oracle as O
    dev = torch.device("cuda:0")
    row0, rows = moa.lift_rows(m, world, rank)
    C_full = torch.full((m, p), float("nan"), dtype=torch.float64, device=dev)
    q_out.put(C_full)                      # CUDA IPC handle to the peer
    peer = q_in.get(timeout=120)           # the peer's C_full, mapped here
    A = torch.from_numpy(I.host_matrix(rows, n, 5, I.ID_A, row0=row0)).to(dev)
    B = torch.from_numpy(I.host_matrix(n, p, 5, I.ID_B)).to(dev)
    barrier.wait()                         # entry barrier: both copies allocated and initialised
    moa.gemm_scatter(A, B, C_full[row0:row0 + rows], [peer[row0:row0 + rows].data_ptr()])
    torch.cuda.synchronize()
    barrier.wait()                         # exit barrier: both epilogues complete
    ref = O.ip(I.host_matrix(m, n, 5, I.ID_A), I.host_matrix(n, p, 5, I.ID_B), fused=True)
    result.put((rank, bool(np.array_equal(C_full.cpu().numpy(), ref))))
    barrier.wait()                         # keep our C_full alive until the peer has checked


@pytest.mark.gpu
def test_scatter_two_process_gather_over_cuda_ipc(cuda_device):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    m, n, p = 1000, 96, 520                # G = 2: rows 500 + 500, ragged tile edges
    q01, q10, res = ctx.Queue(), ctx.Queue(), ctx.Queue()
    bar = ctx.Barrier(2)
    procs = [ctx.Process(target=_ipc_worker, args=(0, 2, m, n, p, q01, q10, bar, res)),
             ctx.Process(target=_ipc_worker, args=(1, 2, m, n, p, q10, q01, bar, res))]
    for pr in procs:
        pr.start()
    out = dict(res.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert out == {0: True, 1: True}


@pytest.mark.gpu
def test_lifted_cols_and_2d_fused_gather_single_rank(cuda_device):
    """Column lifting (Fig. 5 ip_cols.c at GPU level) with C_full in a symmetric window:
    the column block is computed straight into C_full's columns (row stride p) by the
    PEER epilogue path, no workspace; C_full and C_local bitwise moa_gemm."""
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        for (m, n, p) in [(1000, 256, 300), (2000, 48, 2000), (257, 33, 131)]:
            A, B = _operands(m, n, p, 11, cuda_device)
            ref = moa.gemm(A, B)
            C_full = comm.alloc_window((m, p))
            C_full.fill_(float("nan"))
            C_local = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
            moa.gemm_lifted_cols(A, B, C_local, p, comm, C_full=C_full)
            torch.cuda.synchronize()
            assert torch.equal(C_full, ref) and torch.equal(C_local, ref), (m, n, p)
            # 2-D lifting on a 1 x 1 grid through the fused-gather entry
            C_full.fill_(float("nan"))
            C_blk = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
            moa.gemm_lifted_2d(m, p, 1, 1, A, B, C_blk, comm, C_full=C_full)
            torch.cuda.synchronize()
            assert torch.equal(C_full, ref) and torch.equal(C_blk, ref), (m, n, p)
            comm.free_window(C_full)
    finally:
        comm.close()
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,offsets", [(torch.float64, [1]), (torch.float32, [1, 2, 3])])
def test_scatter_destination_not_16B_aligned(cuda_device, dtype, offsets):
    """Regression (round-1 review): a destination aligned to its element but not to 16
    bytes (fp64 at base+8; fp32 at base+4/+8/+12) on a TMA-eligible shape used to
    select K1/K3, whose epilogue stores 16-byte vectors: a misaligned-address fault.
    Such a destination now routes the call to the generic kernel; every destination
    and C hold the oracle's bits."""
    m, n, p = 256, 64, 192                       # TMA-eligible: the chooser would pick K1 / K3
    npdt = np.float64 if dtype == torch.float64 else np.float32
    Ah = I.host_matrix(m, n, 4, I.ID_A, dtype=npdt)
    Bh = I.host_matrix(n, p, 4, I.ID_B, dtype=npdt)
    ref = O.ip(Ah, Bh, fused=True)
    A, B = torch.from_numpy(Ah).to(cuda_device), torch.from_numpy(Bh).to(cuda_device)
    for off in offsets:
        C = torch.full((m, p), float("nan"), dtype=dtype, device=cuda_device)
        buf = torch.full((m * p + 8,), float("nan"), dtype=dtype, device=cuda_device)
        dst = buf[off:off + m * p].view(m, p)       # element-aligned, not 16-B aligned
        assert dst.data_ptr() % 16 != 0
        moa.gemm_scatter(A, B, C, [dst])
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), ref), off
        assert np.array_equal(dst.cpu().numpy(), ref), off
