"""Pins for the CPU oracle (oracle/), run on the dev box (-m "not gpu").

The oracle is pinned to things OTHER than itself: hand-derived worked examples
(tests/golden/, [TRIVIAL]/[DERIVED]), closed forms (delta, tone, constant), invariants
(Parseval, linearity, circular shift, Hermitian symmetry, inverse(forward) = id),
the non-separable brute-force sum on tiny inputs, an independent library (numpy.fft,
numpy float64 matmul), exact integer arithmetic, and matrices with exactly known products
(identity, permutation, Sylvester-Hadamard, orthonormal DCT-II -- P:153 "orthogonal").
Each test names the mistake it would catch.
"""
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    sec, data = None, {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line in ("input", "output"):
                sec = line
                data[sec] = []
                continue
            v = [float(t) for t in line.split()]
            data[sec].append([complex(v[2 * i], v[2 * i + 1]) for i in range(len(v) // 2)])
    return {k: np.array(v, dtype=np.complex128) for k, v in data.items()}


def _rand_c(n0, n1, seed=0):
    r = np.random.default_rng(seed)
    return r.uniform(-1, 1, (n0, n1)) + 1j * r.uniform(-1, 1, (n0, n1))


# ----------------------------------------------------------------------------- FFT pins

def test_worked_2x2():
    """Hand-derived 2x2 example (golden/fft2d_2x2.txt). Catches a wrong sign only via
    ordering of outputs, a transposed result, a missing term."""
    g = _read_golden("fft2d_2x2.txt")
    X = oracle.dft2d(g["input"])
    assert np.array_equal(X, g["output"])


def test_delta_4x4_golden():
    """4x4 delta at (1,1) -> (-i)^(k0+k1) (golden/fft2d_4x4_delta11.txt). Catches a
    sign error (would give (+i)^(k0+k1)) and a transposed index."""
    g = _read_golden("fft2d_4x4_delta11.txt")
    x = np.zeros((4, 4), np.complex128)
    x[1, 1] = 1
    assert np.allclose(oracle.dft2d(x), g["output"], atol=1e-15, rtol=0)


@pytest.mark.parametrize("n0,n1,a,b", [(8, 8, 3, 5), (16, 4, 7, 1), (4, 32, 2, 29), (1, 16, 0, 9),
                                       (32, 1, 17, 0), (64, 64, 63, 1), (6, 10, 5, 7)])
def test_delta_closed_form(n0, n1, a, b):
    """Delta at (a,b) -> exp(-2 pi i (k0 a/N0 + k1 b/N1)). Catches sign, index swap
    (a with b), and wrong modular reduction."""
    x = np.zeros((n0, n1), np.complex128)
    x[a, b] = 1
    k0 = np.arange(n0)[:, None]
    k1 = np.arange(n1)[None, :]
    ref = np.exp(-2j * np.pi * ((k0 * a % n0) / n0 + (k1 * b % n1) / n1))
    assert np.allclose(oracle.dft2d(x), ref, atol=1e-13, rtol=0)


@pytest.mark.parametrize("n0,n1,f0,f1", [(16, 16, 3, 11), (32, 8, 31, 0), (8, 64, 1, 63), (64, 32, 20, 7)])
def test_single_tone(n0, n1, f0, f1):
    """x = exp(+2 pi i (f0 n0/N0 + f1 n1/N1)) -> X = N0 N1 at (f0,f1), 0 elsewhere."""
    i0 = np.arange(n0)[:, None]
    i1 = np.arange(n1)[None, :]
    x = np.exp(2j * np.pi * ((f0 * i0 % n0) / n0 + (f1 * i1 % n1) / n1))
    ref = np.zeros((n0, n1), np.complex128)
    ref[f0, f1] = n0 * n1
    assert np.allclose(oracle.dft2d(x), ref, atol=1e-10 * n0 * n1, rtol=0)
    # and the inverse maps the spike back to the tone (scaling 1/(N0 N1) pinned here)
    assert np.allclose(oracle.dft2d(ref, inverse=True), x, atol=1e-12, rtol=0)


def test_constant():
    x = np.full((8, 16), 0.25 - 0.5j)
    ref = np.zeros((8, 16), np.complex128)
    ref[0, 0] = (0.25 - 0.5j) * 128
    assert np.allclose(oracle.dft2d(x), ref, atol=1e-13, rtol=0)


@pytest.mark.parametrize("n0,n1", [(16, 16), (8, 32), (3, 5), (1, 64), (64, 1)])
def test_numpy_fft2(n0, n1):
    """Independent library (numpy pocketfft, complex128). Catches any systematic error."""
    x = _rand_c(n0, n1, seed=n0 * 100 + n1)
    assert oracle.rel_l2(oracle.dft2d(x), np.fft.fft2(x)) < 1e-14
    assert oracle.rel_l2(oracle.dft2d(x, inverse=True), np.fft.ifft2(x)) < 1e-14


def test_one_row_is_textbook_1d_dft():
    """n0 = 1 reduces the 2D definition to the 1D DFT (numpy.fft.fft)."""
    x = _rand_c(1, 128, seed=3)
    assert oracle.rel_l2(oracle.dft2d(x)[0], np.fft.fft(x[0])) < 1e-14


@pytest.mark.parametrize("n0,n1", [(4, 4), (8, 4), (2, 16), (6, 3)])
def test_bruteforce_nonseparable(n0, n1):
    """Separable evaluation equals the non-separable quadruple sum (definition)."""
    x = _rand_c(n0, n1, seed=7)
    for inv in (False, True):
        assert oracle.rel_l2(oracle.dft2d(x, inv), oracle.dft2d_bruteforce(x, inv)) < 1e-14


def test_parseval_linearity_shift_hermitian_roundtrip():
    n0, n1 = 32, 16
    x = _rand_c(n0, n1, seed=11)
    y = _rand_c(n0, n1, seed=12)
    X = oracle.dft2d(x)
    # Parseval: sum |X|^2 = N sum |x|^2 (catches a wrong scale / dropped term)
    assert np.isclose(np.sum(np.abs(X) ** 2), n0 * n1 * np.sum(np.abs(x) ** 2), rtol=1e-13)
    # Linearity
    a, b = 0.3 - 1.1j, -2.0 + 0.5j
    assert oracle.rel_l2(oracle.dft2d(a * x + b * y), a * X + b * oracle.dft2d(y)) < 1e-14
    # Circular shift: x[n - s] -> X[k] exp(-2 pi i k.s/N)  (catches a transposed index)
    s0, s1 = 5, 3
    xs = np.roll(np.roll(x, s0, axis=0), s1, axis=1)
    k0 = np.arange(n0)[:, None]
    k1 = np.arange(n1)[None, :]
    ph = np.exp(-2j * np.pi * ((k0 * s0 % n0) / n0 + (k1 * s1 % n1) / n1))
    assert oracle.rel_l2(oracle.dft2d(xs), X * ph) < 1e-13
    # Hermitian symmetry for real input
    xr = x.real.copy()
    XR = oracle.dft2d(xr)
    XRm = np.conj(XR[(-k0) % n0, (-k1) % n1])
    assert oracle.rel_l2(XR, XRm) < 1e-14
    # inverse(forward) = identity
    assert oracle.rel_l2(oracle.dft2d(X, inverse=True), x) < 1e-14


def test_sampled_lines_match_full():
    """Sampled output row/column functions agree with the full transform."""
    n0, n1 = 32, 64
    x = synth.complex_field(n0, n1)  # complex64 input path (exact promotion)
    X = oracle.dft2d(x)
    for k1 in (0, 1, 33, 63):
        assert np.allclose(oracle.dft2d_col(x, k1), X[:, k1], rtol=0, atol=1e-12)
    for k0 in (0, 5, 31):
        assert np.allclose(oracle.dft2d_row(x, k0), X[k0, :], rtol=0, atol=1e-12)
    Xi = oracle.dft2d(x, inverse=True)
    assert np.allclose(oracle.dft2d_col(x, 7, inverse=True), Xi[:, 7], rtol=0, atol=1e-14)
    assert np.allclose(oracle.dft2d_row(x, 9, inverse=True), Xi[9, :], rtol=0, atol=1e-14)


def test_f32_input_is_exact_promotion():
    x = synth.complex_field(16, 16)
    assert np.array_equal(oracle.dft2d(x), oracle.dft2d(x.astype(np.complex128)))


# -------------------------------------------------------------------------- matmul pins

def test_identity_and_permutation_exact():
    r = np.random.default_rng(5)
    A = r.uniform(-1, 1, (37, 53))
    assert np.array_equal(oracle.matmul(A, np.eye(53)), A)
    assert np.array_equal(oracle.matmul(np.eye(37), A), A)
    p = r.permutation(37)
    P = np.eye(37)[p]
    assert np.array_equal(oracle.matmul(P, A), A[p])  # catches a transposed operand


@pytest.mark.parametrize("n", [64, 128])
def test_hadamard_exact(n):
    """Sylvester-Hadamard: H H^T = n I exactly (integer partial sums)."""
    H = synth.hadamard(n)
    assert np.array_equal(oracle.matmul(H, np.ascontiguousarray(H.T)), n * np.eye(n))


@pytest.mark.parametrize("n", [64, 256])
def test_dct_orthogonal(n):
    """Orthonormal DCT-II (an orthogonal matrix): Q Q^T = I."""
    Q = synth.dct2_matrix(n)
    assert np.abs(oracle.matmul(Q, np.ascontiguousarray(Q.T)) - np.eye(n)).max() < 1e-13


@pytest.mark.parametrize("m,n,k", [(7, 5, 9), (1, 1, 1), (3, 17, 2), (16, 1, 33)])
def test_small_integer_exact(m, n, k):
    """Brute force in exact Python integers (catches dropped terms, wrong index)."""
    r = np.random.default_rng(m * n * k)
    A = r.integers(-8, 9, (m, k))
    B = r.integers(-8, 9, (k, n))
    ref = [[sum(int(A[i, p]) * int(B[p, j]) for p in range(k)) for j in range(n)] for i in range(m)]
    assert np.array_equal(oracle.matmul(A.astype(np.float64), B.astype(np.float64)),
                          np.array(ref, dtype=np.float64))


def test_numpy_matmul_and_strides():
    r = np.random.default_rng(9)
    A = r.uniform(-1, 1, (65, 130))
    B = r.uniform(-1, 1, (130, 47))
    assert oracle.rel_l2(oracle.matmul(A, B), A @ B) < 1e-14
    # leading dimensions larger than the logical width (views)
    Abig = r.uniform(-1, 1, (65, 160))
    Bbig = r.uniform(-1, 1, (130, 64))
    Av, Bv = Abig[:, :130], Bbig[:, :47]
    assert oracle.rel_l2(oracle.matmul(Av, Bv), Av @ Bv) < 1e-14


def test_matmul_rows_cols_match_full():
    A = synth.real_matrix(40, 70, synth.TID_GEMM_A)
    B = synth.real_matrix(70, 50, synth.TID_GEMM_B)
    C = oracle.matmul(A, B)
    rows = [0, 13, 39]
    cols = [0, 1, 49]
    assert np.array_equal(oracle.matmul_rows(A, B, rows), C[rows])
    assert np.array_equal(oracle.matmul_cols(A, B, cols), C[:, cols].T)
    # f32 path is an exact promotion of the f64 path
    assert np.array_equal(C, oracle.matmul(A.astype(np.float64), B.astype(np.float64)))


# ------------------------------------------------------------------------ input recipe

def test_synth_recipe():
    a = synth.uniform_pm1(1000, 1)
    assert np.array_equal(a, synth.uniform_pm1(1000, 1))
    assert a.min() >= -1 and a.max() < 1
    # global indexing: a shard equals the matching slice of the whole
    full = synth.complex_field(16, 32)
    part = synth.complex_field(16, 32, row0=5, rows=4)
    assert np.array_equal(full[5:9], part)
    # values are exact multiples of 2^-23 (FP32-exact) and mostly not TF32-exact
    v = a.astype(np.float64) * 2 ** 23
    assert np.array_equal(v, np.round(v))
    bits = a.view(np.uint32) & 0x1FFF
    assert np.mean(bits != 0) > 0.9


# ---------------------------------------------------------------- batched 1D DFT (N4)
def test_dft1d_rows_hand_and_closed_forms():
    """n = 2 by hand ([a, b] -> [a + b, a - b]); delta at t0 -> exp(-2 pi i k t0 / n); a
    single tone exp(+2 pi i f t / n) -> n at k = f; inverse o forward = identity."""
    x = np.array([[1 + 2j, 3 - 1j], [0.5, -0.25j]], dtype=np.complex64)
    X = oracle.dft1d_rows(x)
    assert np.allclose(X, [[4 + 1j, -2 + 3j], [0.5 - 0.25j, 0.5 + 0.25j]], atol=1e-15)
    n = 64
    k = np.arange(n)
    d = np.zeros((3, n), dtype=np.complex64)
    for b, t0 in enumerate((0, 5, 63)):
        d[b, t0] = 1
    D = oracle.dft1d_rows(d)
    for b, t0 in enumerate((0, 5, 63)):
        assert np.allclose(D[b], np.exp(-2j * np.pi * k * t0 / n), atol=1e-14)
    f = 7
    tone = np.exp(2j * np.pi * f * k / n)[None, :]
    T = oracle.dft1d_rows(tone)
    ref = np.zeros(n, dtype=complex)
    ref[f] = n
    assert np.abs(T[0] - ref).max() < 1e-12
    x = synth.complex_field(5, 32)
    assert oracle.rel_l2(oracle.dft1d_rows(oracle.dft1d_rows(x), inverse=True), x) < 1e-14


def test_dft1d_rows_vs_numpy():
    x = synth.complex_field(9, 128)
    assert oracle.rel_l2(oracle.dft1d_rows(x), np.fft.fft(x.astype(np.complex128), axis=1)) < 1e-14
    assert oracle.rel_l2(oracle.dft1d_rows(x, inverse=True), np.fft.ifft(x.astype(np.complex128), axis=1)) < 1e-14
