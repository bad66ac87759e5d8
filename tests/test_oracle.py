"""Pins for the CPU oracle (run without a GPU: ``-m "not gpu"``).

Each test ties ``oracle/`` to something other than itself: exact rational
arithmetic within the classical error bound, an independent step-by-step brute
force with exactly-rounded steps, integer exactness, algebraic identities,
closed forms, library routines (numpy) and the worked examples in
``tests/golden/`` (each with its citation). A plausible slip in the oracle (a
dropped term, a wrong index or stride, a transposed operand, a wrong loop
order, a fused/unfused mix-up) fails at least one of them.
"""
from __future__ import annotations

import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
U64 = 2.0 ** -53
U32 = 2.0 ** -24


def _rand(rng, m, n, dtype):
    return rng.uniform(-1.0, 1.0, size=(m, n)).astype(dtype)


def _round_f32(x: Fraction) -> np.float32:
    """Correctly rounded (RN-even) Fraction -> float32, avoiding double rounding."""
    f = np.float32(float(x))
    best = f
    for cand in (np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))):
        dc, db = abs(Fraction(float(cand)) - x), abs(Fraction(float(best)) - x)
        if dc < db or (dc == db and (int(cand.view(np.uint32)) & 1) == 0):
            best = cand
    return np.float32(best)


def _brute(A, B, fused: bool):
    """Independent brute force: for every (i, j), k ascending, each step rounded
    exactly once (fused: round(a*b + s) via exact rationals) or twice (unfused:
    round(round(a*b) + s), native IEEE arithmetic which Python never contracts)."""
    m, n = A.shape
    p = B.shape[1]
    f32 = A.dtype == np.float32
    C = np.zeros((m, p), dtype=A.dtype)
    for i in range(m):
        for j in range(p):
            s = A.dtype.type(0)
            for k in range(n):
                a, b = A[i, k], B[k, j]
                if fused:
                    ex = Fraction(float(a)) * Fraction(float(b)) + Fraction(float(s))
                    s = _round_f32(ex) if f32 else np.float64(float(ex))
                else:
                    s = A.dtype.type(s + A.dtype.type(a * b))
            C[i, j] = s
    return C


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("fused", [False, True])
def test_exact_rational_within_higham_bound(dtype, fused):
    """|C_oracle - C_exact| <= gamma_n (|A||B|) elementwise (Higham, recursive summation).
    A dropped term, wrong index, or transposed operand breaks this by O(|a b|)."""
    rng = np.random.default_rng(11)
    u = U64 if dtype == np.float64 else U32
    for trial in range(40):
        m, n, p = rng.integers(1, 8, size=3)
        A, B = _rand(rng, m, n, dtype), _rand(rng, n, p, dtype)
        C = O.ip(A, B, fused=fused)
        gamma = n * u / (1 - n * u)
        absAB = np.abs(A.astype(np.float64)) @ np.abs(B.astype(np.float64))
        for i in range(m):
            for j in range(p):
                exact = sum(Fraction(float(A[i, k])) * Fraction(float(B[k, j])) for k in range(n))
                err = abs(Fraction(float(C[i, j])) - exact)
                assert err <= Fraction(gamma) * Fraction(float(absAB[i, j])) * (1 + 1e-12), (trial, i, j)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("fused", [False, True])
def test_bruteforce_exact_steps_bitwise(dtype, fused):
    """ip.c (i-sigma-j) == independent per-(i,j) brute force with k ascending, bit for bit."""
    rng = np.random.default_rng(12 + int(fused))
    for shape in [(1, 1, 1), (3, 5, 4), (7, 9, 6), (9, 2, 9), (4, 13, 3)]:
        m, n, p = shape
        A, B = _rand(rng, m, n, dtype), _rand(rng, n, p, dtype)
        C = O.ip(A, B, fused=fused)
        ref = _brute(A, B, fused)
        assert np.array_equal(C.view(np.uint8), ref.view(np.uint8)), shape


def test_fused_and_unfused_differ_on_random_data():
    """R3 matters: the two readings are distinguishable (guards against both names
    silently binding the same routine)."""
    rng = np.random.default_rng(5)
    A, B = _rand(rng, 32, 64, np.float64), _rand(rng, 64, 32, np.float64)
    assert not np.array_equal(O.ip(A, B, fused=False), O.ip(A, B, fused=True))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("fused", [False, True])
def test_integer_valued_exact(dtype, fused):
    """Integer-valued inputs: every partial sum is an exactly representable integer,
    so the oracle must equal exact integer matrix multiplication (Python ints)."""
    rng = np.random.default_rng(3)
    for (m, n, p) in [(17, 33, 9), (64, 50, 70), (1, 200, 1)]:
        Ai = rng.integers(-4, 5, size=(m, n))
        Bi = rng.integers(-4, 5, size=(n, p))
        exact = np.array([[sum(int(Ai[i, k]) * int(Bi[k, j]) for k in range(n)) for j in range(p)] for i in range(m)])
        C = O.ip(Ai.astype(dtype), Bi.astype(dtype), fused=fused)
        assert np.array_equal(C, exact.astype(dtype))


def test_worked_examples_golden():
    with open(os.path.join(GOLDEN, "gemm_worked_examples.json")) as f:
        g = json.load(f)
    for c in g["cases"]:
        for dtype in (np.float64, np.float32):
            for fused in (False, True):
                A = np.array(c["A"], dtype=dtype).reshape(c["m"], c["n"])
                B = np.array(c["B"], dtype=dtype).reshape(c["n"], c["p"])
                C = O.ip(A, B, fused=fused)
                assert np.array_equal(C.ravel(), np.array(c["C"], dtype=dtype)), c["name"]


@pytest.mark.parametrize("fused", [False, True])
def test_identities_bitwise(fused):
    """A•I = A, I•B = B, A•0 = 0 exactly; (A•B)^T = B^T•A^T bitwise (products
    commute exactly and the sigma order is the same)."""
    rng = np.random.default_rng(4)
    m, n, p = 23, 31, 19
    A, B = _rand(rng, m, n, np.float64), _rand(rng, n, p, np.float64)
    assert np.array_equal(O.ip(A, np.eye(n), fused=fused), A)
    assert np.array_equal(O.ip(np.eye(m), A, fused=fused), A)
    assert np.array_equal(O.ip(A, np.zeros((n, p)), fused=fused), np.zeros((m, p)))
    C = O.ip(A, B, fused=fused)
    Ct = O.ip(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T), fused=fused)
    assert np.array_equal(C.T, Ct)


def test_rank1_closed_form():
    """A = u v^T, B = w z^T (integers) => C_ij = u_i z_j (v·w) exactly."""
    rng = np.random.default_rng(6)
    m, n, p = 40, 57, 33
    u, z = rng.integers(-2, 3, size=m), rng.integers(-2, 3, size=p)
    v, w = rng.integers(-1, 2, size=n), rng.integers(-1, 2, size=n)
    A, B = np.outer(u, v).astype(np.float64), np.outer(w, z).astype(np.float64)
    C = O.ip(A, B)
    assert np.array_equal(C, np.outer(u, z).astype(np.float64) * float(v @ w))
    ones = O.ip(np.ones((5, 77)), np.ones((77, 6)))
    assert np.all(ones == 77.0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_matches_numpy_matmul_within_tolerance(dtype):
    """Library routine (numpy/BLAS, different summation order) agrees within the
    north_star tolerance on a non-square, non-symmetric case; a transposed operand
    or swapped m/p would be far outside it."""
    rng = np.random.default_rng(7)
    A, B = _rand(rng, 37, 129, dtype), _rand(rng, 129, 53, dtype)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    tol = 1e-12 if dtype == np.float64 else 1e-5
    for fused in (False, True):
        C = O.ip(A, B, fused=fused).astype(np.float64)
        rel = np.linalg.norm(C - ref) / np.linalg.norm(ref)
        assert rel <= tol * np.sqrt(129)


def test_transposed_operand_is_detected():
    """Sanity that the pins are sharp: a transposed B gives a clearly different C."""
    rng = np.random.default_rng(8)
    A, B = _rand(rng, 16, 16, np.float64), _rand(rng, 16, 16, np.float64)
    ref = A @ B
    bad = O.ip(A, np.ascontiguousarray(B.T))
    assert np.linalg.norm(bad - ref) / np.linalg.norm(ref) > 0.1


@pytest.mark.parametrize("fused", [False, True])
def test_lifting_listings_bitwise(fused):
    """Fig. 4 ip_rows.c and Fig. 5 ip_cols.c are re-indexings of ip.c: bitwise equal
    (S:366). ip_rows with np = m (one row per processor) and np = 1 too."""
    rng = np.random.default_rng(9)
    m, n, p = 24, 37, 16
    A, B = _rand(rng, m, n, np.float64), _rand(rng, n, p, np.float64)
    C = O.ip(A, B, fused=fused)
    for np_ in (1, 2, 3, 4, 8, 24):
        assert np.array_equal(O.ip_rows(A, B, np_, fused=fused), C)
    A32, B32 = A.astype(np.float32), B.astype(np.float32)
    assert np.array_equal(O.ip_rows(A32, B32, 4, fused=fused), O.ip(A32, B32, fused=fused))
    if not fused:
        for rsize in (1, 2, 4, 8, 16):
            assert np.array_equal(O.ip_cols(A, B, rsize), C)
    with pytest.raises(ValueError):
        O.ip_rows(A, B, 5)
    with pytest.raises(ValueError):
        O.ip_cols(A, B, 3)


def test_classical_ijk_equals_onf_bitwise():
    """Row-times-column and ONF i-sigma-j perform the same rounding sequence
    per element (k ascending, unfused): bitwise equal on random floats."""
    rng = np.random.default_rng(10)
    for dtype in (np.float64, np.float32):
        A, B = _rand(rng, 31, 45, dtype), _rand(rng, 45, 27, dtype)
        assert np.array_equal(O.ip_ijk(A, B), O.ip(A, B))


def test_row_subsets_bitwise():
    rng = np.random.default_rng(13)
    m, n, p = 50, 21, 30
    A, B = _rand(rng, m, n, np.float64), _rand(rng, n, p, np.float64)
    for fused in (False, True):
        C = O.ip(A, B, fused=fused)
        rows = [0, m - 1, 7, 7, 31]
        assert np.array_equal(O.ip_rows_subset(A, B, rows, fused=fused), C[rows])
        assert np.array_equal(O.ip_rowblock(A[10:20], B, fused=fused), C[10:20])
    with pytest.raises(IndexError):
        O.ip_rows_subset(A, B, [m])


def test_f32_truth_is_double_accumulation():
    rng = np.random.default_rng(14)
    A, B = _rand(rng, 9, 40, np.float32), _rand(rng, 40, 11, np.float32)
    T = O.ip_f32_truth(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.max(np.abs(T - ref)) < 1e-13


def test_empty_extents():
    for (m, n, p) in [(0, 3, 4), (3, 0, 4), (3, 4, 0), (0, 0, 0)]:
        C = O.ip(np.ones((m, n)), np.ones((n, p)))
        assert C.shape == (m, p) and np.all(C == 0)


# ---------------- shapes, psi, lifting, paper-mode block arithmetic ----------------

def test_psi_gamma_golden():
    with open(os.path.join(GOLDEN, "psi_examples.json")) as f:
        g = json.load(f)
    for c in g["gamma"]:
        if c["shape"]:
            assert O.gamma_row(c["idx"], c["shape"]) == c["offset"], c
        else:
            assert O.psi([], []) == (0, 1)
    for c in g["psi"]:
        off, cnt = O.psi(c["idx"], c["shape"])
        assert c["data"][off:off + cnt] == c["result"], c


def test_psi_matches_numpy_indexing_and_identity():
    """Bracket bridge rav(i psi xi) == (rav xi)[gamma] checked against numpy basic
    indexing (library), for all prefixes of random shapes; psi identity
    (iota(rho xi)) psi xi == xi."""
    rng = random.Random(1)
    for _ in range(60):
        rank = rng.randint(1, 4)
        shape = [rng.randint(1, 5) for _ in range(rank)]
        X = np.arange(int(np.prod(shape))).reshape(shape)
        for q in range(rank + 1):
            idx = [rng.randrange(s) for s in shape[:q]]
            off, cnt = O.psi(idx, shape)
            assert np.array_equal(X.ravel()[off:off + cnt], np.ravel(X[tuple(idx)]))
        rebuilt = [X.ravel()[O.psi(list(ix), shape)[0]] for ix in np.ndindex(*shape)]
        assert np.array_equal(np.array(rebuilt).reshape(shape), X)
    with pytest.raises(IndexError):
        O.psi([3], [3, 4])
    with pytest.raises(IndexError):
        O.psi([0, 0, 0], [3, 4])


def test_lift_rows_balanced_and_reduces_to_listing():
    for m in range(0, 70):
        for G in range(1, 10):
            parts = [O.lift_rows(m, G, g) for g in range(G)]
            assert sum(r for _, r in parts) == m
            assert parts[0][0] == 0
            for g in range(1, G):
                assert parts[g][0] == parts[g - 1][0] + parts[g - 1][1]
            assert max(r for _, r in parts) - min(r for _, r in parts) <= 1
            if m % G == 0:  # Fig. 4: processor k owns i = ip + (sizel/np)*k, ip < sizel/np
                for k, (r0, r) in enumerate(parts):
                    assert (r0, r) == ((m // G) * k, m // G)
    with pytest.raises(ValueError):
        O.lift_rows(10, 0, 0)
    with pytest.raises(ValueError):
        O.lift_rows(10, 2, 2)


def test_paper_block_arithmetic_golden():
    with open(os.path.join(GOLDEN, "paper_block_arithmetic.json")) as f:
        g = json.load(f)
    e = g["elem_bytes"]
    for c in g["cases"]:
        b = O.select_block_paper(c["l1_budget_bytes"], e)
        assert b == c["block_side"]
        assert b * b * e == c["bytes_per_block"]
        assert 3 * b * b * e == c["total_bytes_3_blocks"]
        assert 3 * (2 * b) ** 2 * e > c["l1_budget_bytes"]  # maximal
    for r, c in g["equal_count_shapes_1024"]:
        assert r * c == 32 * 32
    assert O.select_block_paper(24, 8) == 1
    with pytest.raises(ValueError):
        O.select_block_paper(23, 8)
