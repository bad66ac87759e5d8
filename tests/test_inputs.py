"""The seeded input generator (inputs/): deterministic, in range, row-block
consistent, and — on the GPU — bit-identical between host and device."""
import numpy as np
import pytest

from inputs import inputs as I


def test_host_deterministic_and_in_range():
    a = I.host_matrix(64, 33, seed=1, mid=I.ID_A)
    b = I.host_matrix(64, 33, seed=1, mid=I.ID_A)
    assert np.array_equal(a, b)
    assert a.min() >= -1.0 and a.max() < 1.0
    assert abs(a.mean()) < 0.1 and 0.25 < a.var() < 0.42  # uniform[-1,1): var 1/3
    c = I.host_matrix(64, 33, seed=2, mid=I.ID_A)
    d = I.host_matrix(64, 33, seed=1, mid=I.ID_B)
    assert not np.array_equal(a, c) and not np.array_equal(a, d)


def test_host_uniform_values_are_exact_dyadics():
    a = I.host_matrix(16, 16, seed=3, mid=I.ID_A)
    scaled = (a + 1.0) * 2.0 ** 52
    assert np.array_equal(scaled, np.floor(scaled))
    f = I.host_matrix(16, 16, seed=3, mid=I.ID_A, dtype=np.float32)
    s32 = (f.astype(np.float64) + 1.0) * 2.0 ** 23
    assert np.array_equal(s32, np.floor(s32))


def test_int_kind():
    a = I.host_matrix(100, 50, seed=4, mid=I.ID_B, kind=I.INT)
    assert set(np.unique(a)).issubset(set(range(-4, 5)))
    assert len(np.unique(a)) == 9


def test_row_blocks_match_full_matrix():
    full = I.host_matrix(40, 17, seed=5, mid=I.ID_A)
    part = I.host_matrix(7, 17, seed=5, mid=I.ID_A, row0=13)
    assert np.array_equal(full[13:20], part)
    rows = I.host_rows([0, 39, 5], 17, seed=5, mid=I.ID_A)
    assert np.array_equal(rows, full[[0, 39, 5]])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind", [I.UNIFORM, I.INT])
def test_device_generator_matches_host_bitwise(cuda_device, dtype, kind):
    import torch
    tdt = torch.float64 if dtype == "f64" else torch.float32
    ndt = np.float64 if dtype == "f64" else np.float32
    for (rows, cols, row0) in [(1, 1, 0), (37, 129, 0), (300, 512, 1000)]:
        t = torch.empty((rows, cols), dtype=tdt, device=cuda_device)
        I.device_fill(t, seed=9, mid=I.ID_B, kind=kind, row0=row0)
        h = I.host_matrix(rows, cols, seed=9, mid=I.ID_B, kind=kind, dtype=ndt, row0=row0)
        assert np.array_equal(t.cpu().numpy().view(np.uint8), h.view(np.uint8))
