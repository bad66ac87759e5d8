"""CUDA-graph capture of the C-ABI calls (the B200 way to amortise launch cost of
small, repeated GEMMs): the very FIRST call of a fresh process happens inside
stream capture, so every one-time setup of the library (device query, pools,
kernel attributes) must be capture-safe. Replays must equal the oracle bitwise,
including plans that use the tile counter (memset node) and the stream-K flags
(self-resetting, reused by every replay)."""
from __future__ import annotations

import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = textwrap.dedent(r'''
    import sys, numpy as np, torch
    sys.path.insert(0, ".")
    import paper_2306_11148_b200 as moa
    from inputs import inputs as I
    from oracle import oracle as O
    # (m, n, p): latency tiles; stream-K runs only (tiles < 2 grid); dynamic + runs
    shapes = [(256, 256, 256), (2000, 96, 2000), (4096, 48, 4096)]
    host = [(I.host_matrix(m, n, 7, I.ID_A), I.host_matrix(n, p, 7, I.ID_B)) for (m, n, p) in shapes]
    dev = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in host]
    outs = [torch.full((a.shape[0], b.shape[1]), float("nan"), dtype=torch.float64, device="cuda") for a, b in dev]
    # and the fused-gather epilogue (K1 PEER) into a second block
    sc = torch.full_like(outs[1], float("nan"))
    sd = torch.full_like(outs[1], float("nan"))
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):   # first library calls of this process
            for (a, b), c in zip(dev, outs):
                moa.gemm(a, b, out=c)
            moa.gemm_scatter(dev[1][0], dev[1][1], sc, [sd])
    torch.cuda.synchronize()
    for rep in range(3):
        for c in outs + [sc, sd]:
            c.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for (a, b), c in zip(host, outs):
            assert np.all(c.cpu().numpy() == O.ip(a, b, fused=True)), ("replay", rep, a.shape, b.shape)
        assert torch.equal(sc, outs[1]) and torch.equal(sd, outs[1]), ("scatter replay", rep)
    print("GRAPH OK")
''')


def test_first_call_inside_graph_capture(cuda_device):
    r = subprocess.run([sys.executable, "-c", SCRIPT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "GRAPH OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
