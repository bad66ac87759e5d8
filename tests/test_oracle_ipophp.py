"""Pins for the ipophp-sibling oracles (Hadamard, Kronecker): SPEC worked examples,
numpy (library, exact: one rounding per element), algebraic laws — the
mixed-product property ties Kronecker to the GEMM oracle."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_golden():
    g = json.load(open(os.path.join(GOLDEN, "ipophp_examples.json")))
    for dt in (np.float64, np.float32):
        for c in g["hadamard"]:
            A = np.array(c["A"], dt).reshape(c["m"], c["n"])
            B = np.array(c["B"], dt).reshape(c["m"], c["n"])
            assert np.array_equal(O.hadamard(A, B).ravel(), np.array(c["C"], dt))
        for c in g["kron"]:
            A = np.array(c["A"], dt).reshape(c["m"], c["n"])
            B = np.array(c["B"], dt).reshape(c["p"], c["q"])
            assert np.array_equal(O.kron(A, B).ravel(), np.array(c["C"], dt))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_against_numpy_bitwise(dt):
    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, (13, 17)).astype(dt)
    B = rng.uniform(-1, 1, (13, 17)).astype(dt)
    assert np.array_equal(O.hadamard(A, B), A * B)
    K = rng.uniform(-1, 1, (5, 3)).astype(dt)
    L = rng.uniform(-1, 1, (4, 7)).astype(dt)
    assert np.array_equal(O.kron(K, L), np.kron(K, L))


def test_kron_laws():
    rng = np.random.default_rng(2)
    A, B = rng.integers(-3, 4, (3, 4)).astype(np.float64), rng.integers(-3, 4, (2, 5)).astype(np.float64)
    Cm, D = rng.integers(-3, 4, (4, 2)).astype(np.float64), rng.integers(-3, 4, (5, 3)).astype(np.float64)
    # mixed product: (A (x) B)(C (x) D) = (AC) (x) (BD), exact on integers, via the GEMM oracle
    lhs = O.ip(O.kron(A, B), O.kron(Cm, D))
    rhs = O.kron(O.ip(A, Cm), O.ip(B, D))
    assert np.array_equal(lhs, rhs)
    assert np.array_equal(O.kron(A, B).T, O.kron(np.ascontiguousarray(A.T), np.ascontiguousarray(B.T)))
    assert np.array_equal(O.kron(np.ones((1, 1)), B), B)
    assert np.array_equal(O.hadamard(A, np.ones_like(A)), A)
    assert np.array_equal(O.hadamard(A, B[:, :4][:2].repeat(2, 0)[:3]), O.hadamard(B[:, :4][:2].repeat(2, 0)[:3], A))
