"""Pins for the GEMM oracle (oracle/gemm.py): closed forms, exact integer
products, identities and a brute-force sum -- none of them re-uses the
oracle's own matmul call."""
import numpy as np
import pytest

from oracle import gemm_abt, gemm_abt_rows, gemm_loops


def test_brute_force_tiny():
    rng = np.random.default_rng(0)
    A, B = rng.standard_normal((5, 7)), rng.standard_normal((3, 7))
    np.testing.assert_allclose(gemm_abt(A, B), gemm_loops(A, B), rtol=1e-13, atol=1e-13)


def test_identity_and_permutation():
    """A I^T = A; a permutation matrix B picks and reorders columns of A."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((6, 4))
    np.testing.assert_array_equal(gemm_abt(A, np.eye(4)), A)
    perm = [2, 0, 3, 1]
    P = np.eye(4)[perm]          # row n of P is e_{perm[n]}
    np.testing.assert_array_equal(gemm_abt(A, P), A[:, perm])


def test_orientation_is_abt_not_ab():
    """C[m, n] pairs row m of A with ROW n of B (B is [N, K], K-contiguous)."""
    A = np.array([[1.0, 2.0, 3.0]])
    B = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    np.testing.assert_array_equal(gemm_abt(A, B), [[1.0, 3.0]])


def test_exact_small_integers():
    """Integer-valued inputs: every partial sum is an exactly representable integer."""
    rng = np.random.default_rng(2)
    A = rng.integers(-8, 9, size=(64, 96)).astype(np.float64)
    B = rng.integers(-8, 9, size=(48, 96)).astype(np.float64)
    ref = np.array([[int(sum(int(a) * int(b) for a, b in zip(A[m], B[n]))) for n in range(48)] for m in range(64)])
    np.testing.assert_array_equal(gemm_abt(A, B), ref)


def test_rank_one_closed_form():
    """A = u 1^T, B = v 1^T -> C = K u v^T."""
    u, v, K = np.array([1.0, -2.0, 0.5]), np.array([3.0, 4.0]), 10
    C = gemm_abt(np.outer(u, np.ones(K)), np.outer(v, np.ones(K)))
    np.testing.assert_allclose(C, K * np.outer(u, v), rtol=0, atol=0)


def test_rows_helper_matches():
    rng = np.random.default_rng(3)
    A, B = rng.standard_normal((9, 5)), rng.standard_normal((4, 5))
    np.testing.assert_allclose(gemm_abt_rows(A, B, [0, 8, 3]), gemm_loops(A, B)[[0, 8, 3]], rtol=1e-13)


def test_bad_shapes():
    with pytest.raises(ValueError):
        gemm_abt(np.zeros((2, 3)), np.zeros((2, 4)))
