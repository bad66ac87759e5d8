"""Row-lifted (multi-processor) path: Fig. 4 ip_rows.c.

CPU (`-m "not gpu"`): world_size-2 gloo processes exercise the host logic of
moa_gemm_lifted — the 128-byte id exchange (Comm.exchange_unique_id), the row
partition from the C ABI (moa_lift_rows), the broadcast of B from rank 0, the
per-rank compute of its rows (oracle here — no GPU) and the gather of C in
partition order — and check the assembled C equals the single-process oracle
bit for bit (lifting is a re-indexing).
GPU: a 1-rank NCCL communicator drives the real moa_gemm_lifted (broadcast,
lifted compute, gather) and must equal moa_gemm bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, n, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_11148_b200 as moa
        from inputs import inputs as I
        from oracle import oracle as O
        uid = moa.Comm.exchange_unique_id(make_id=lambda: bytes(range(128)))
        assert uid == bytes(range(128))
        row0, rows = moa.lift_rows(m, world, rank)
        A_local = I.host_matrix(rows, n, 3, I.ID_A, row0=row0)
        B = torch.from_numpy(I.host_matrix(n, p, 3, I.ID_B)) if rank == 0 else torch.zeros((n, p), dtype=torch.float64)
        dist.broadcast(B, src=0)  # the lifted path's one exchange (reading R13)
        C_local = torch.from_numpy(O.ip_rowblock(A_local, B.numpy(), fused=True))
        counts = [moa.lift_rows(m, world, g)[1] for g in range(world)]
        parts = [torch.zeros((c, p), dtype=torch.float64) for c in counts]
        dist.all_gather(parts, C_local) if len(set(counts)) == 1 else _gather_uneven(parts, C_local, rank, world)
        if rank == 0:
            C = torch.cat(parts).numpy()
            A = I.host_matrix(m, n, 3, I.ID_A)
            q.put(bool(np.array_equal(C, O.ip(A, B.numpy(), fused=True))))
    finally:
        dist.destroy_process_group()


def _gather_uneven(parts, mine, rank, world):
    for g in range(world):
        buf = mine if g == rank else parts[g]
        dist.broadcast(buf, src=g)
        if g == rank:
            parts[g].copy_(mine)


@pytest.mark.parametrize("m", [64, 37])
def test_lifted_host_logic_gloo_world2(m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, 24, 40, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    ok = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert ok


@pytest.mark.gpu
def test_lifted_nccl_single_rank_equals_gemm(cuda_device):
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        for (m, n, p) in [(1000, 256, 300), (129, 64, 128)]:
            A = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
            B = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
            I.device_fill(A, 5, I.ID_A)
            I.device_fill(B, 5, I.ID_B)
            ref = moa.gemm(A, B)
            C_local = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
            C_full = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
            moa.gemm_lifted(m, A, B, C_local, comm, C_full=C_full)
            torch.cuda.synchronize()
            assert torch.equal(C_local, ref) and torch.equal(C_full, ref)
    finally:
        comm.close()
        dist.destroy_process_group()


@pytest.mark.gpu
def test_lifted_pipelined_panels_single_rank(cuda_device):
    """NEXT-1 step 1: the k-panel pipelined exchange path (side stream, per-panel events,
    accumulate launches) gives the one-launch bits. Exercised here with one rank and
    explicit npanels (the broadcast itself is a no-op with one rank)."""
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        m, n, p = 700, 1000, 300
        A = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
        B = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
        I.device_fill(A, 6, I.ID_A)
        I.device_fill(B, 6, I.ID_B)
        ref = moa.gemm(A, B)
        for K in (1, 2, 3, 5, 16):
            C = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
            moa.gemm_lifted(m, A, B, C, comm, npanels=K)
            torch.cuda.synchronize()
            assert torch.equal(C, ref), K
    finally:
        comm.close()
        dist.destroy_process_group()



def _worker_cols(rank, world, port, m, n, p, q):
    """Column lifting (Fig. 5 ip_cols.c across processes): rank g computes C[:, cols_g]
    from all of A (broadcast) and its column block of B; the gathered C equals the
    single-process oracle bit for bit."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_11148_b200 as moa
        from inputs import inputs as I
        from oracle import oracle as O
        c0, cg = moa.lift_rows(p, world, rank)
        A = torch.from_numpy(I.host_matrix(m, n, 4, I.ID_A)) if rank == 0 else torch.zeros((m, n), dtype=torch.float64)
        dist.broadcast(A, src=0)
        B = I.host_matrix(n, p, 4, I.ID_B)
        C_local = torch.from_numpy(O.ip(A.numpy(), np.ascontiguousarray(B[:, c0:c0 + cg]), fused=True))
        blocks = [torch.zeros((m, moa.lift_rows(p, world, g)[1]), dtype=torch.float64) for g in range(world)]
        for g in range(world):
            buf = C_local if g == rank else blocks[g]
            dist.broadcast(buf, src=g)
            if g == rank:
                blocks[g].copy_(C_local)
        if rank == 0:
            C = torch.cat(blocks, dim=1).numpy()
            q.put(bool(np.array_equal(C, O.ip(A.numpy(), B, fused=True))))
    finally:
        dist.destroy_process_group()


def test_column_lifting_host_logic_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cols, args=(r, 2, port, 20, 16, 37, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    ok = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert ok


@pytest.mark.gpu
def test_lifted_cols_nccl_single_rank(cuda_device):
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        m, n, p = 300, 128, 260
        A = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
        B = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
        I.device_fill(A, 7, I.ID_A)
        I.device_fill(B, 7, I.ID_B)
        ref = moa.gemm(A, B)
        C_local = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
        C_full = torch.full((m, p), float("nan"), dtype=torch.float64, device=cuda_device)
        moa.gemm_lifted_cols(A, B, C_local, p, comm, C_full=C_full)
        torch.cuda.synchronize()
        assert torch.equal(C_local, ref) and torch.equal(C_full, ref)
    finally:
        comm.close()
        dist.destroy_process_group()



def _worker_2d(rank, world, port, gr, gc, m, n, p, q):
    """2-D lifting on a gr x gc process grid (gloo): A row panels travel along process
    rows, B column panels along process columns; the assembled C equals the oracle."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2306_11148_b200 as moa
        from inputs import inputs as I
        from oracle import oracle as O
        r, c = rank // gc, rank % gc
        r0, rows = moa.lift_rows(m, gr, r)
        c0, cols = moa.lift_rows(p, gc, c)
        groups_r = [dist.new_group([i * gc + j for j in range(gc)]) for i in range(gr)]
        groups_c = [dist.new_group([i * gc + j for i in range(gr)]) for j in range(gc)]
        A_panel = torch.from_numpy(I.host_matrix(rows, n, 5, I.ID_A, row0=r0)) if c == 0 else torch.zeros((rows, n), dtype=torch.float64)
        Bfull = I.host_matrix(n, p, 5, I.ID_B)
        B_panel = torch.from_numpy(np.ascontiguousarray(Bfull[:, c0:c0 + cols])) if r == 0 else torch.zeros((n, cols), dtype=torch.float64)
        dist.broadcast(A_panel, src=r * gc, group=groups_r[r])
        dist.broadcast(B_panel, src=c, group=groups_c[c])
        C_block = torch.from_numpy(O.ip(A_panel.numpy(), B_panel.numpy(), fused=True))
        gathered = [None] * world if rank == 0 else None
        dist.gather_object((r0, rows, c0, cols, C_block.numpy()), gathered, dst=0)
        if rank == 0:
            C = np.full((m, p), np.nan)
            for (a, ra, b, cb, blk) in gathered:
                C[a:a + ra, b:b + cb] = blk
            A = I.host_matrix(m, n, 5, I.ID_A)
            q.put(bool(np.array_equal(C, O.ip(A, Bfull, fused=True))))
    finally:
        dist.destroy_process_group()


def test_2d_lifting_host_logic_gloo_2x2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, 4, port, 2, 2, 21, 12, 19, q)) for r in range(4)]
    for pr in procs:
        pr.start()
    ok = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert ok


@pytest.mark.gpu
def test_lifted_2d_nccl_single_rank(cuda_device):
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        m, n, p = 200, 96, 136
        A = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
        B = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
        I.device_fill(A, 8, I.ID_A)
        I.device_fill(B, 8, I.ID_B)
        C = torch.empty((m, p), dtype=torch.float64, device=cuda_device)
        moa.gemm_lifted_2d(m, p, 1, 1, A, B, C, comm)
        torch.cuda.synchronize()
        assert torch.equal(C, moa.gemm(A, B))
        with pytest.raises(moa.MoAError):
            moa.gemm_lifted_2d(m, p, 2, 1, A, B, C, comm)  # grid does not match the rank count
    finally:
        comm.close()
        dist.destroy_process_group()


@pytest.mark.gpu
def test_lifted_host_pipeline_single_rank(cuda_device):
    """moa_gemm_lifted_host: the e2e pipeline with B's k-panels broadcast from rank 0
    on the communicator's side stream (1-rank NCCL: the broadcasts run, as no-ops)
    gives moa_gemm's bits, with and without the first-panel k-chain."""
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(_free_port()))
        dist.init_process_group("gloo", rank=0, world_size=1)
    comm = moa.Comm(device=0)
    try:
        # (1000 x 1000: n >= 512 but too few rows for a row-panel split — with a
        #  communicator it still chains over the 8 B k-panels every rank broadcasts)
        for (m, n, p) in [(6400, 640, 384), (300, 200, 100), (1000, 1000, 130), (0, 640, 64)]:
            A = torch.empty((m, n), dtype=torch.float64, device=cuda_device)
            B = torch.empty((n, p), dtype=torch.float64, device=cuda_device)
            if m:
                I.device_fill(A, 4, I.ID_A)
            I.device_fill(B, 4, I.ID_B)
            ref = moa.gemm(A, B).cpu()
            hA, hB = A.cpu().pin_memory(), B.cpu().pin_memory()
            hC = torch.full((m, p), float("nan"), dtype=torch.float64).pin_memory()
            Ad, Bd, Cd = torch.empty_like(A), torch.zeros_like(B), torch.empty((m, p), dtype=torch.float64,
                                                                                device=cuda_device)
            moa.gemm_lifted_host(m, hA, hB, hC, Ad, Bd, Cd, comm)
            assert torch.equal(hC, ref), (m, n, p)
    finally:
        comm.close()
        dist.destroy_process_group()
