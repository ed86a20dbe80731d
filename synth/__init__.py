"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no DFT, no matrix product).  It only
draws numbers.  Both sides of every parity test (oracle/ and the CUDA path) receive
the same host arrays produced here, so neither side generates its own inputs.

Recipe:

* SEED = 200409883 (the arXiv id).
* seed_t = mix64(SEED ^ tensor_id)                  (one stream per tensor)
* value(i) = (top24(mix64(seed_t + i)) - 2**23) / 2**23  in [-1, 1)
  where i is the GLOBAL row-major element index (complex: re uses 2i, im uses 2i+1),
  so a shard, the full array and the oracle all see identical values.
  These values are exact in FP32 and, in general, NOT exact in TF32, so the
  3xTF32 lo path of the GEMM is exercised.
* mix64 is the SplitMix64 finaliser applied to (x + golden gamma).

Structured sets that mirror the paper's workloads ("vibration frequency
analysis", "orthogonal matrix data"):

* ``tones2d``: a sum of integer-frequency 2D complex tones plus small uniform noise.
* ``dct2_matrix``: the orthonormal DCT-II matrix Q (Q Q^T = I), an orthogonal matrix.
* ``hadamard``: the Sylvester-Hadamard matrix H[i,j] = (-1)^popcount(i&j).
"""
from __future__ import annotations

import numpy as np

SEED = 200409883
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 22

# tensor ids (stable across the repo so that stored fixtures stay valid)
TID_FFT_X = 1
TID_GEMM_A = 2
TID_GEMM_B = 3
TID_NOISE = 4


def mix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 output function of (x + gamma), elementwise on uint64 (wrapping)."""
    with np.errstate(over="ignore"):
        z = x + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _mix64_scalar(x: int) -> int:
    return int(mix64(np.array([x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def stream_seed(tensor_id: int, seed: int = SEED) -> int:
    return _mix64_scalar((seed ^ tensor_id) & 0xFFFFFFFFFFFFFFFF)


def uniform_pm1(count: int, tensor_id: int, start: int = 0, seed: int = SEED,
                out: np.ndarray | None = None) -> np.ndarray:
    """float32 values in [-1,1) for global indices [start, start+count)."""
    st = np.uint64(stream_seed(tensor_id, seed))
    if out is None:
        out = np.empty(count, dtype=np.float32)
    for c0 in range(0, count, _CHUNK):
        c1 = min(count, c0 + _CHUNK)
        with np.errstate(over="ignore"):
            idx = np.arange(start + c0, start + c1, dtype=np.uint64) + st
        u = (mix64(idx) >> np.uint64(40)).astype(np.int64)  # top 24 bits
        out[c0:c1] = (u - (1 << 23)).astype(np.float32) * np.float32(2.0 ** -23)
    return out


def uniform_pm1_f64(count: int, tensor_id: int, start: int = 0, seed: int = SEED) -> np.ndarray:
    """float64 values in [-1,1) with a FULL 53-bit mantissa draw (top 53 bits of the same
    SplitMix64 stream): products of two such values are not exact in FP64, so an FP64 GEMM
    test on them probes the rounding of every product, not only the accumulation order."""
    st = np.uint64(stream_seed(tensor_id, seed))
    out = np.empty(count, dtype=np.float64)
    for c0 in range(0, count, _CHUNK):
        c1 = min(count, c0 + _CHUNK)
        with np.errstate(over="ignore"):
            idx = np.arange(start + c0, start + c1, dtype=np.uint64) + st
        u = (mix64(idx) >> np.uint64(11)).astype(np.int64)  # top 53 bits
        out[c0:c1] = (u - (1 << 52)).astype(np.float64) * 2.0 ** -52
    return out


def real_matrix_f64(m: int, n: int, tensor_id: int, seed: int = SEED) -> np.ndarray:
    """m x n float64 matrix of full-mantissa values in [-1, 1) (see uniform_pm1_f64)."""
    return uniform_pm1_f64(m * n, tensor_id, seed=seed).reshape(m, n)


def complex_field(n0: int, n1: int, tensor_id: int = TID_FFT_X, row0: int = 0,
                  rows: int | None = None, seed: int = SEED) -> np.ndarray:
    """complex64 [rows, n1] slice (rows row0..row0+rows) of the global n0 x n1 field."""
    rows = n0 - row0 if rows is None else rows
    flat = uniform_pm1(2 * rows * n1, tensor_id, start=2 * row0 * n1, seed=seed)
    return flat.view(np.complex64).reshape(rows, n1)


def real_matrix(m: int, n: int, tensor_id: int, row0: int = 0, rows: int | None = None,
                dtype=np.float32, seed: int = SEED) -> np.ndarray:
    """[rows, n] slice of the global m x n matrix with values in [-1,1)."""
    rows = m - row0 if rows is None else rows
    a = uniform_pm1(rows * n, tensor_id, start=row0 * n, seed=seed).reshape(rows, n)
    return a.astype(dtype, copy=False)


def tones2d(n0: int, n1: int, ntones: int = 8, noise: float = 1e-3,
            seed: int = SEED) -> tuple[np.ndarray, list[tuple[int, int, complex]]]:
    """Paper-flavoured FFT input (P:149 vibration analysis): integer 2D tones + noise.

    Returns (complex64 field, [(f0, f1, amplitude), ...]).  Frequencies are drawn from
    the seeded stream so the set is reproducible.
    """
    rng = uniform_pm1(4 * ntones, TID_NOISE, seed=seed ^ 0x5A5A)
    tones = []
    for t in range(ntones):
        f0 = int((rng[4 * t] * 0.5 + 0.5) * n0) % n0
        f1 = int((rng[4 * t + 1] * 0.5 + 0.5) * n1) % n1
        amp = complex(float(rng[4 * t + 2]), float(rng[4 * t + 3]))
        tones.append((f0, f1, amp))
    i0 = np.arange(n0, dtype=np.int64)[:, None]
    i1 = np.arange(n1, dtype=np.int64)[None, :]
    x = np.zeros((n0, n1), dtype=np.complex128)
    for f0, f1, amp in tones:
        # exact integer phase reduction before the angle is formed
        ph = ((f0 * i0) % n0) / n0 + ((f1 * i1) % n1) / n1
        x += amp * np.exp(2j * np.pi * ph)
    x += noise * complex_field(n0, n1, TID_NOISE, seed=seed).astype(np.complex128)
    return x.astype(np.complex64), tones


def dct2_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II matrix Q[k, j] (float64); Q @ Q.T == I (P:153 'orthogonal')."""
    k = np.arange(n, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    q = np.sqrt(2.0 / n) * np.cos(np.pi * (2.0 * j + 1.0) * k / (2.0 * n))
    q[0, :] = np.sqrt(1.0 / n)
    return q


def hadamard(n: int, row0: int = 0, rows: int | None = None) -> np.ndarray:
    """Sylvester-Hadamard rows H[row0:row0+rows, :] as float32 (entries +-1)."""
    rows = n - row0 if rows is None else rows
    i = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    j = np.arange(n, dtype=np.uint64)[None, :]
    b = i & j
    par = np.zeros(b.shape, dtype=np.uint64)
    while np.any(b):
        par ^= b & np.uint64(1)
        b = b >> np.uint64(1)
    return (1.0 - 2.0 * par.astype(np.float32)).astype(np.float32)
