"""The lifted paths' exchange plan (moa_exchange_plan) against the byte model — CPU.

Row lifting (Fig. 4 ip_rows.c): every processor reads all of B (B carries
no processor index), so B (n·p elements) reaches every rank once; the optional
gather of C (reading R14) moves m·p elements in total. Column lifting (Fig. 5
ip_cols.c): A (m·n) reaches every rank once. 2-D lifting: A's row
panel travels along each process row, B's column panel along each process column.
SURVEY §8(d)/(e) gives these byte counts; the plan must match them exactly, issue the
same sequence on every rank of a communicator, and be empty on one rank. The GPU test
tests/test_lifted_multiproc_gpu.py checks that the executors issue exactly this plan.
"""
from __future__ import annotations

import itertools

import pytest

import paper_2306_11148_b200 as moa

F64, F32 = moa.F64, moa.F32


def _plans(variant, m, n, p, G, **kw):
    return [moa.exchange_plan(variant, m, n, p, kw.get("dtype", F64), G, r, kw.get("gr", 0), kw.get("gc", 0),
                              kw.get("npanels", 0), kw.get("flags", 0)) for r in range(G)]


def _nccl(ops, comm=None):
    return [(o.op, o.comm, o.root, o.count, o.offset, o.group) for o in ops
            if o.op != "pull" and (comm is None or o.comm == comm)]


SHAPES = [(300, 96, 200), (301, 160, 136), (2, 64, 96), (32768, 32768, 32768), (65536, 512, 512), (0, 64, 64),
          (64, 0, 64), (64, 64, 0), (1000, 1, 3)]


@pytest.mark.parametrize("m,n,p", SHAPES)
@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("npanels", [0, 1, 3])
def test_rows_broadcast_moves_B_once_and_is_rank_identical(m, n, p, G, npanels):
    plans = _plans(moa.XPLAN_ROWS, m, n, p, G, npanels=npanels)
    if G == 1:
        assert plans == [[]]
        return
    assert all(_nccl(pl) == _nccl(plans[0]) for pl in plans)
    b = [o for o in plans[0] if o.operand == "B"]
    assert all(o.op == "broadcast" and o.root == 0 and o.phase == 1 for o in b)
    assert sum(o.count for o in b) == n * p
    # contiguous k-panels in ascending order (MoA order: each one byte range of B)
    off = 0
    for o in b:
        assert o.offset == off and o.count >= 0
        off += o.count
    # panel 0 on the full communicator; later panels on the CTA-limited pipe split
    assert all((o.comm == "world") == (o.panel == 0) for o in b)
    if npanels > 0 and n * p > 0:
        assert max(o.panel for o in b) <= npanels - 1


@pytest.mark.parametrize("m,n,p", SHAPES)
@pytest.mark.parametrize("G", [2, 3, 4, 8])
def test_rows_gather_moves_C_once(m, n, p, G):
    plans = _plans(moa.XPLAN_ROWS, m, n, p, G, flags=moa.XF_GATHER)
    assert all(_nccl(pl) == _nccl(plans[0]) for pl in plans)
    c = [o for o in plans[0] if o.operand == "C"]
    if m * p == 0:
        assert c == []
        return
    if m % G == 0:
        assert len(c) == 1 and c[0].op == "allgather" and c[0].count * G == m * p
    else:  # one broadcast per rank with rows, rooted at that rank, in one NCCL group
        rows = [moa.lift_rows(m, G, g) for g in range(G)]
        assert [(o.root, o.offset, o.count) for o in c] == [(g, r0 * p, rg * p) for g, (r0, rg) in enumerate(rows) if rg]
        assert len({o.group for o in c}) == 1 and c[0].group > 0
    assert all(o.phase == 2 for o in c)


@pytest.mark.parametrize("m,n,p", SHAPES)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_rows_pull_reads_B_once_per_rank(m, n, p, G):
    for flags in (moa.XF_PULL_B, moa.XF_PULL_B | moa.XF_FUSED_GATHER):
        plans = _plans(moa.XPLAN_ROWS, m, n, p, G, flags=flags)
        # the NCCL part (two barriers) is identical on every rank
        assert all(_nccl(pl) == _nccl(plans[0]) for pl in plans)
        if m * p == 0 and n * p == 0:
            assert plans[0] == []
            continue
        assert [o.op for o in plans[0] if o.op != "pull"] == ["barrier", "barrier"]
        assert not [o for o in plans[0] if o.op == "pull"]  # rank 0 owns B
        for r in range(1, G):
            pulls = [o for o in plans[r] if o.op == "pull"]
            assert sum(o.count for o in pulls) == n * p
            assert all(o.root == 0 and o.phase == 1 for o in pulls)
            assert [o.panel for o in pulls] == list(range(len(pulls)))


@pytest.mark.parametrize("m,n,p,G", [(4096, 4096, 4096, 8), (100, 64, 50, 3), (0, 64, 64, 2), (64, 64, 64, 1)])
def test_rows_direct_moves_no_B(m, n, p, G):
    """NEXT-1 step 2 (moa_gemm_lifted_direct): B never travels as a collective or a copy —
    the plan is the entry and exit barrier around rank 0's window, identical on every
    rank, plus the optional NCCL gather of C."""
    for gather in (0, moa.XF_GATHER):
        plans = _plans(moa.XPLAN_ROWS, m, n, p, G, flags=moa.XF_DIRECT_B | gather)
        assert all(pl == plans[0] for pl in plans)
        if G == 1 or (m * p == 0 and n * p == 0):
            assert plans[0] == []
            continue
        assert not [o for o in plans[0] if o.operand == "B" or o.op == "pull"]
        ops = [o.op for o in plans[0]]
        assert ops[0] == "barrier" and ops[-1] == "barrier"
        assert (len(ops) > 2) == bool(gather and m * p > 0)


def test_pull_panels_geometric():
    for n in [0, 1, 31, 63, 64, 100, 512, 4096, 16384, 32768, 65536, 10 ** 6]:
        b = moa.pull_panels(n)
        assert b[0] == 0 and b[-1] == n and len(b) - 1 <= 16
        assert all(x < y for x, y in zip(b, b[1:])) or n == 0
        assert all(x % 32 == 0 for x in b[:-1])
        if n >= 64:
            first = b[1]
            assert first == max(32, (n // 64) // 32 * 32)
            # each panel (but the last) at most doubles the rows available before it
            for j in range(2, len(b) - 1):
                assert b[j] - b[j - 1] <= b[j - 1]
    assert moa.pull_panels(32768) == [0, 512, 1024, 2048, 4096, 8192, 16384, 32768]


@pytest.mark.parametrize("m,n,p", SHAPES)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_host_plan_moves_B_once(m, n, p, G):
    plans = _plans(moa.XPLAN_ROWS_HOST, m, n, p, G)
    assert all(_nccl(pl) == _nccl(plans[0]) for pl in plans)
    assert sum(o.count for o in plans[0]) == n * p
    # one broadcast per B k-panel: 8 (16 for deep k, n >= 24576), none split when n < 512
    assert len(plans[0]) <= ((16 if n >= 24576 else 8) if n >= 512 else 1)


@pytest.mark.parametrize("m,n,p", SHAPES)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_cols_moves_A_exactly_once(m, n, p, G):
    for flags in (0, moa.XF_GATHER, moa.XF_FUSED_GATHER):
        plans = _plans(moa.XPLAN_COLS, m, n, p, G, flags=flags)
        assert all(_nccl(pl) == _nccl(plans[0]) for pl in plans)
        a = [o for o in plans[0] if o.operand == "A"]
        assert len(a) == (1 if m * n > 0 else 0)  # round 1 broadcast A twice on the fused path
        if a:
            assert (a[0].op, a[0].root, a[0].count) == ("broadcast", 0, m * n)
        c = [o for o in plans[0] if o.operand == "C" and o.op == "broadcast"]
        if flags == moa.XF_GATHER and m * p > 0:
            assert sum(o.count for o in c) == m * p
            assert [o.root for o in c] == [g for g in range(G) if moa.lift_rows(p, G, g)[1] > 0]
        else:
            assert c == []
        if flags == moa.XF_FUSED_GATHER:
            assert [o.op for o in plans[0]].count("barrier") == 2


@pytest.mark.parametrize("m,n,p", [(257, 96, 131), (64, 32, 200), (1, 8, 1), (32768, 32768, 32768)])
@pytest.mark.parametrize("gr,gc", [(1, 2), (2, 1), (2, 2), (2, 4), (4, 2), (1, 8)])
def test_2d_moves_panels_along_rows_and_columns(m, n, p, gr, gc):
    G = gr * gc
    for flags in (0, moa.XF_FUSED_GATHER):
        plans = _plans(moa.XPLAN_2D, m, n, p, G, gr=gr, gc=gc, flags=flags)
        for r, c in itertools.product(range(gr), range(gc)):
            ops = plans[r * gc + c]
            _, rows = moa.lift_rows(m, gr, r)
            _, cols = moa.lift_rows(p, gc, c)
            a = [o for o in ops if o.operand == "A"]
            b = [o for o in ops if o.operand == "B"]
            assert [(o.comm, o.root, o.count) for o in a] == ([("row", 0, rows * n)] if gc > 1 and rows * n else [])
            assert [(o.comm, o.root, o.count) for o in b] == ([("col", 0, n * cols)] if gr > 1 and n * cols else [])
            # same ops as every other rank of its process row / column
            assert _nccl(ops, "row") == _nccl(plans[r * gc], "row")
            assert _nccl(ops, "col") == _nccl(plans[c], "col")
            assert _nccl(ops, "world") == _nccl(plans[0], "world")


def test_plan_argument_errors():
    with pytest.raises(moa.MoAError):
        moa.exchange_plan(moa.XPLAN_2D, 8, 8, 8, F64, 4, 0, 3, 1)
    with pytest.raises(moa.MoAError):
        moa.exchange_plan(9, 8, 8, 8, F64, 2, 0)
    with pytest.raises(moa.MoAError):
        moa.exchange_plan(moa.XPLAN_ROWS, -1, 8, 8, F64, 2, 0)
    with pytest.raises(moa.MoAError):
        moa.exchange_plan(moa.XPLAN_ROWS, 8, 8, 8, F64, 2, 2)
    # more ops than the caller's array: the needed count is reported
    ops = moa.exchange_plan(moa.XPLAN_COLS, 64, 64, 1000, F64, 100, 0, flags=moa.XF_GATHER)
    assert len(ops) == 101  # (the binding retried with the reported size)
