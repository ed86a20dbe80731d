"""ctypes wrapper around oracle/liboracle.so (the plain CPU oracle, see oracle.h).

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs.  The product package paper_2004_09883_b200 never
imports this module; the two share no code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lib = None

IN_F64 = 0
IN_F32 = 1


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, OpenMP, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", _SO + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, i64, ci, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.oracle_dft2d.argtypes = [vp, ci, dp, i64, i64, ci, ci]
        L.oracle_dft2d_bruteforce.argtypes = [vp, ci, dp, i64, i64, ci]
        L.oracle_dft1d_rows.argtypes = [vp, ci, dp, i64, i64, ci, ci]
        L.oracle_dft2d_col.argtypes = [vp, ci, i64, i64, i64, ci, dp, ci]
        L.oracle_dft2d_row.argtypes = [vp, ci, i64, i64, i64, ci, dp, ci]
        L.oracle_matmul.argtypes = [i64, i64, i64, vp, i64, vp, i64, ci, dp, i64, ci]
        L.oracle_matmul_rows.argtypes = [i64, i64, i64, vp, i64, vp, i64, ci, vp, i64, dp, ci]
        L.oracle_matmul_cols.argtypes = [i64, i64, i64, vp, i64, vp, i64, ci, vp, i64, dp, ci]
        L.oracle_threads.argtypes = [ci]
        L.oracle_lu.argtypes = [i64, vp, i64, vp, ci]
        for f in ("oracle_dft2d", "oracle_dft2d_bruteforce", "oracle_dft1d_rows", "oracle_dft2d_col",
                  "oracle_dft2d_row", "oracle_matmul", "oracle_matmul_rows",
                  "oracle_matmul_cols", "oracle_threads", "oracle_lu"):
            getattr(L, f).restype = ci
        _lib = L
    return _lib


def threads(n: int = 0) -> int:
    return lib().oracle_threads(n)


def _cin(x):
    """Complex input -> (contiguous array, in_type) without changing its values."""
    x = np.asarray(x)
    if x.dtype == np.complex64:
        return np.ascontiguousarray(x), IN_F32
    return np.ascontiguousarray(x, dtype=np.complex128), IN_F64


def _rin(a):
    a = np.asarray(a)
    if a.dtype == np.float32:
        return a, IN_F32
    return a.astype(np.float64, copy=False), IN_F64


def _check(rc, name):
    if rc != 0:
        raise RuntimeError(f"{name} failed with code {rc}")


def dft2d(x, inverse: bool = False, nthreads: int = 0) -> np.ndarray:
    """2D DFT definition; complex128 result.  inverse scales by 1/(n0 n1)."""
    x, t = _cin(x)
    n0, n1 = x.shape
    X = np.empty((n0, n1), dtype=np.complex128)
    _check(lib().oracle_dft2d(x.ctypes.data, t, X.ctypes.data, n0, n1,
                              1 if inverse else -1, nthreads), "oracle_dft2d")
    return X


def dft1d_rows(x, inverse: bool = False, nthreads: int = 0) -> np.ndarray:
    """1D DFT definition of every row of x[batch][n] (inverse scales by 1/n)."""
    x, t = _cin(x)
    b, n = x.shape
    X = np.empty((b, n), dtype=np.complex128)
    _check(lib().oracle_dft1d_rows(x.ctypes.data, t, X.ctypes.data, b, n, 1 if inverse else -1, nthreads),
           "oracle_dft1d_rows")
    return X


def dft2d_bruteforce(x, inverse: bool = False) -> np.ndarray:
    x, t = _cin(x)
    n0, n1 = x.shape
    X = np.empty((n0, n1), dtype=np.complex128)
    _check(lib().oracle_dft2d_bruteforce(x.ctypes.data, t, X.ctypes.data, n0, n1,
                                         1 if inverse else -1), "oracle_dft2d_bruteforce")
    return X


def dft2d_col(x, k1: int, inverse: bool = False, nthreads: int = 0) -> np.ndarray:
    x, t = _cin(x)
    n0, n1 = x.shape
    out = np.empty(n0, dtype=np.complex128)
    _check(lib().oracle_dft2d_col(x.ctypes.data, t, n0, n1, k1, 1 if inverse else -1,
                                  out.ctypes.data, nthreads), "oracle_dft2d_col")
    return out


def dft2d_row(x, k0: int, inverse: bool = False, nthreads: int = 0) -> np.ndarray:
    x, t = _cin(x)
    n0, n1 = x.shape
    out = np.empty(n1, dtype=np.complex128)
    _check(lib().oracle_dft2d_row(x.ctypes.data, t, n0, n1, k0, 1 if inverse else -1,
                                  out.ctypes.data, nthreads), "oracle_dft2d_row")
    return out


def _mm_args(A, B):
    A, ta = _rin(A)
    B, tb = _rin(B)
    if ta != tb:
        A, B = A.astype(np.float64), B.astype(np.float64)
        ta = tb = IN_F64
    if A.strides[1] != A.itemsize or B.strides[1] != B.itemsize:
        raise ValueError("row-major operands with unit column stride required")
    return A, B, ta, A.strides[0] // A.itemsize, B.strides[0] // B.itemsize


def matmul(A, B, nthreads: int = 0) -> np.ndarray:
    """C = A B by the triple-loop definition (P:153/P:165 matrix block), float64 result."""
    A, B, t, lda, ldb = _mm_args(A, B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    C = np.empty((m, n), dtype=np.float64)
    _check(lib().oracle_matmul(m, n, k, A.ctypes.data, lda, B.ctypes.data, ldb, t,
                               C.ctypes.data, n, nthreads), "oracle_matmul")
    return C


def matmul_rows(A, B, rows, nthreads: int = 0) -> np.ndarray:
    A, B, t, lda, ldb = _mm_args(A, B)
    m, k = A.shape
    n = B.shape[1]
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    C = np.empty((len(rows), n), dtype=np.float64)
    _check(lib().oracle_matmul_rows(m, n, k, A.ctypes.data, lda, B.ctypes.data, ldb, t,
                                    rows.ctypes.data, len(rows), C.ctypes.data, nthreads),
           "oracle_matmul_rows")
    return C


def matmul_cols(A, B, cols, nthreads: int = 0) -> np.ndarray:
    """Returns C[:, cols].T as an (len(cols), m) array."""
    A, B, t, lda, ldb = _mm_args(A, B)
    m, k = A.shape
    n = B.shape[1]
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    C = np.empty((len(cols), m), dtype=np.float64)
    _check(lib().oracle_matmul_cols(m, n, k, A.ctypes.data, lda, B.ctypes.data, ldb, t,
                                    cols.ctypes.data, len(cols), C.ctypes.data, nthreads),
           "oracle_matmul_cols")
    return C


def rel_l2(y, ref) -> float:
    """||y - ref||_2 / ||ref||_2 over all real components (SURVEY §8(c) error metric)."""
    y = np.asarray(y).astype(np.complex128 if np.iscomplexobj(y) or np.iscomplexobj(ref)
                             else np.float64)
    ref = np.asarray(ref).astype(y.dtype)
    den = np.linalg.norm(ref.ravel())
    num = np.linalg.norm((y - ref).ravel())
    return float(num / den) if den > 0 else float(num)


def lu(A, nthreads: int = 0):
    """P A = L U with partial pivoting (P:153/P:165 LU block). Returns (LU, ipiv, info):
    LU holds unit-lower L below the diagonal and U on/above it; ipiv[k] = row swapped with k."""
    LU = np.array(A, dtype=np.float64, order="C", copy=True)
    n = LU.shape[0]
    assert LU.shape == (n, n)
    ipiv = np.empty(n, dtype=np.int32)
    info = lib().oracle_lu(n, LU.ctypes.data, n, ipiv.ctypes.data, nthreads)
    if info < 0:
        raise RuntimeError("oracle_lu failed")
    return LU, ipiv, info


def lu_permutation(ipiv) -> np.ndarray:
    """Row order p such that (P A)[i] = A[p[i]] for the swap sequence ipiv."""
    p = np.arange(len(ipiv))
    for k, q in enumerate(ipiv):
        p[k], p[q] = p[q], p[k]
    return p
