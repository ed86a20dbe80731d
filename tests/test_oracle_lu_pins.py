"""Pins for the LU oracle (P:153 LU of an orthogonal 2048x2048 matrix; cuSOLVER getrf).

Independent of the oracle's own arithmetic: a hand-derived 3x3 example (golden), exact
rational-arithmetic elimination with the same pivot rule on small integer matrices, LAPACK
dgetrf via scipy (independent library), closed forms (triangular / permutation inputs) and
|det Q| = 1 for the orthogonal DCT-II matrix the paper's workload names."""
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "lu_3x3.txt")


def _golden():
    sec, d = None, {}
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line in ("A", "LU", "IPIV"):
            sec = line
            d[sec] = []
            continue
        d[sec].append(line.split())
    A = np.array([[float(Fraction(t)) for t in r] for r in d["A"]])
    LU = np.array([[float(Fraction(t)) for t in r] for r in d["LU"]])
    ipiv = np.array([int(t) for t in d["IPIV"][0]])
    return A, LU, ipiv


def test_hand_example():
    A, LU_ref, ipiv_ref = _golden()
    LU, ipiv, info = oracle.lu(A)
    assert info == 0
    assert np.array_equal(ipiv, ipiv_ref)
    assert np.allclose(LU, LU_ref, rtol=0, atol=1e-15)


def _exact_lu(A):
    n = len(A)
    M = [[Fraction(int(v)) for v in row] for row in A]
    piv = []
    for k in range(n):
        p = max(range(k, n), key=lambda i: (abs(M[i][k]), -i))  # first max
        piv.append(p)
        M[k], M[p] = M[p], M[k]
        if M[k][k] == 0:
            continue
        for i in range(k + 1, n):
            M[i][k] = M[i][k] / M[k][k]
            for j in range(k + 1, n):
                M[i][j] -= M[i][k] * M[k][j]
    return M, piv


@pytest.mark.parametrize("n,seed", [(4, 1), (6, 2), (8, 3)])
def test_exact_rational(n, seed):
    r = np.random.default_rng(seed)
    A = r.integers(-9, 10, (n, n)).astype(np.float64)
    M, piv = _exact_lu(A)
    LU, ipiv, info = oracle.lu(A)
    assert list(ipiv) == piv
    assert np.allclose(LU, np.array([[float(v) for v in row] for row in M]), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("n", [5, 64, 300])
def test_lapack_dgetrf(n):
    """scipy.linalg.lu_factor = LAPACK dgetrf (column-major; same P A = L U, first-max pivots)."""
    A = synth.real_matrix(n, n, synth.TID_GEMM_A, dtype=np.float64)
    lu_s, piv_s = scipy.linalg.lu_factor(A)
    LU, ipiv, info = oracle.lu(A)
    assert np.array_equal(ipiv, piv_s)
    assert np.abs(LU - lu_s).max() <= 1e-12 * np.abs(lu_s).max()


def test_reconstruction_and_orthogonal_det():
    """P Q = L U and |det Q| = |prod u_ii| = 1 for the orthonormal DCT-II Q."""
    n = 256
    Q = synth.dct2_matrix(n)
    LU, ipiv, info = oracle.lu(Q)
    assert info == 0
    L = np.tril(LU, -1) + np.eye(n)
    U = np.triu(LU)
    p = oracle.lu_permutation(ipiv)
    assert np.abs(Q[p] - L @ U).max() < 1e-13
    assert abs(abs(np.prod(np.diag(U))) - 1.0) < 1e-11


def test_closed_forms():
    # diagonally dominant upper triangular: no swaps, L = I, U = A
    U0 = np.triu(np.arange(1, 26, dtype=np.float64).reshape(5, 5)) + 100 * np.eye(5)
    LU, ipiv, info = oracle.lu(U0)
    assert np.array_equal(ipiv, np.arange(5)) and np.array_equal(LU, U0)
    # permutation matrix: P A = I exactly
    perm = np.array([3, 0, 4, 1, 2])
    P = np.eye(5)[perm]
    LU, ipiv, info = oracle.lu(P)
    assert np.array_equal(LU, np.eye(5))
    assert np.array_equal(P[oracle.lu_permutation(ipiv)], np.eye(5))
    # singular: zero column -> info = k+1, factorisation continues
    S = np.array([[0.0, 1.0], [0.0, 2.0]])
    LU, ipiv, info = oracle.lu(S)
    assert info == 1
