"""C-ABI boundary checks that need no GPU: libfb.so loads, exports every symbol include/fb.h
declares, and rejects invalid arguments synchronously (before touching the device)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "fb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fb_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2004_09883_b200 as fb
    return fb.lib()


def test_exports_every_declared_symbol(L):
    import paper_2004_09883_b200 as fb
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(fb.EXPORTS) == syms


def test_status_strings_and_version(L):
    assert L.fb_version() >= 100
    assert L.fb_status_string(0) == b"FB_OK"
    assert L.fb_status_string(2) == b"FB_ERR_UNSUPPORTED_SIZE"
    assert L.fb_status_string(99) == b"FB_ERR_UNKNOWN"


def test_fft_validation_without_device(L):
    p = ctypes.c_void_p(16)
    # beyond 16384 (power of two) or 8192 (other lengths) -> FB_ERR_UNSUPPORTED_SIZE (2)
    assert L.fb_fft2d(p, p, 8193, 4, None, 0, None) == 2
    assert L.fb_fft2d(p, p, 32768, 4, None, 0, None) == 2
    assert b"power" in L.fb_last_error_detail()
    # other lengths <= 8192 (Bluestein) are accepted and need a workspace (FB_ERR_WORKSPACE, 4)
    assert L.fb_fft2d(p, p, 3, 4, None, 0, None) == 4
    assert L.fb_fft2d_workspace_bytes(3, 4) > 0 and L.fb_fft2d_workspace_bytes(8191, 8192) > 0
    assert L.fb_fft2d_workspace_bytes(8193, 8) == 0
    assert L.fb_fft2d(p, p, 0, 4, None, 0, None) == 1
    assert L.fb_fft2d(None, p, 4, 4, None, 0, None) == 1
    # misaligned
    assert L.fb_fft2d(ctypes.c_void_p(8), p, 4, 4, None, 0, None) == 3
    # partial overlap: x = 16, y = 24 (sizes 128 bytes)
    assert L.fb_ifft2d(ctypes.c_void_p(16), ctypes.c_void_p(32), 4, 4, None, 0, None) == 1
    # workspace rules
    assert L.fb_fft2d_workspace_bytes(256, 256) == 0            # one column pass, in place
    assert L.fb_fft2d_workspace_bytes(2048, 2048) == 2048 * 2048 * 8  # 2 x 1024 split plan
    assert L.fb_fft2d_workspace_bytes(8192, 64) == 8192 * 64 * 8
    assert L.fb_fft2d(p, ctypes.c_void_p(1 << 40), 8192, 64, None, 0, None) == 4
    # streaming host form: batch >= 1, two slots of the fb_fft2d_host scratch, checked before any device work
    one = L.fb_fft2d_host_workspace_bytes(2048, 2048)
    assert L.fb_fft2d_host_batch_workspace_bytes(2048, 2048) == 2 * ((one + 255) // 256 * 256)
    assert L.fb_fft2d_host_batch(p, p, 2048, 2048, 0, 0, p, 1 << 40, None) == 1
    assert L.fb_fft2d_host_batch(p, p, 2048, 10000, 2, 0, p, 1 << 40, None) == 2
    assert L.fb_fft2d_host_batch(p, p, 2048, 2048, 2, 0, p, one, None) == 4


def test_matmul_validation_without_device(L):
    p = ctypes.c_void_p(1 << 20)
    q = ctypes.c_void_p(1 << 30)
    r = ctypes.c_void_p(1 << 35)
    assert L.fb_matmul(2, 4, 4, 4, p, 4, q, 4, r, 4, None, 0, None) == 1        # bad dtype
    assert L.fb_matmul(1, 0, 4, 4, p, 4, q, 4, r, 4, None, 0, None) == 1        # m = 0
    assert L.fb_matmul(1, 4, 4, 4, p, 3, q, 4, r, 4, None, 0, None) == 1        # lda < k
    assert L.fb_matmul(0, 4, 4, 5, p, 5, q, 4, r, 4, None, 0, None) == 3        # lda*4 % 16
    assert L.fb_matmul(1, 4, 4, 4, p, 4, p, 4, p, 4, None, 0, None) == 1        # C aliases A
    assert L.fb_matmul(0, 64, 64, 64, p, 64, q, 64, r, 64, None, 0, None) == 4  # FP32 needs ws
    assert L.fb_matmul_workspace_bytes(1, 64, 64, 64) == 0
    assert L.fb_matmul_workspace_bytes(0, 64, 32, 30) == (2 * 64 * 32 + 2 * 32 * 32) * 4


def test_nr_shim_validation_without_device(L):
    nn = (ctypes.c_ulong * 3)(0, 3, 4)
    data = (ctypes.c_float * 25)()
    assert L.fb_nr_fourn(data, nn, 2, -1) == 2   # 3 is not a power of two
    assert L.fb_nr_fourn(data, nn, 3, -1) == 1   # ndim 3 unsupported
    assert L.fb_nr_fourn(data, nn, 2, 0) == 1    # isign must be +-1


def test_comm_validation_without_device(L):
    assert L.fb_comm_unique_id_bytes() == 128
    p = ctypes.c_void_p(16)
    assert L.fb_fft2d_slab(None, p, p, 16, 16, p, 4096, None) == 5
    assert L.fb_matmul_rowblock(None, 0, 8, 8, 8, p, 8, p, 8, 0, p, 8, None, 0, None) == 5
    assert L.fb_comm_destroy(None) == 0
    assert L.fb_fft2d_slab_workspace_bytes(4, 64, 32) == 2 * 16 * 32 * 8


def test_slab_model_and_fused_query_validation(L):
    p = ctypes.c_void_p(1 << 20)
    assert L.fb_comm_fused(None) == 0
    assert L.fb_comm_fused_detail(None) == b"null communicator"
    assert L.fb_fft2d_slab_model(0, 0, p, p, 64, 64, p, p, 1 << 20, None) == 1   # P < 1
    assert L.fb_fft2d_slab_model(9, 0, p, p, 64, 64, p, p, 1 << 20, None) == 1   # P > 8
    assert L.fb_fft2d_slab_model(4, 0, p, p, 64, 2, p, p, 1 << 20, None) == 2    # n1 % P
    assert L.fb_fft2d_slab_model(2, 0, p, p, 64, 64, p, p, 16, None) == 4        # workspace


def test_fft1d_batched_validation(L):
    p = ctypes.c_void_p(1 << 20)
    assert L.fb_fft1d_batched(p, p, 3, 4, None) == 2        # not a power of two
    assert L.fb_fft1d_batched(p, p, 32768, 4, None) == 2    # > 16384
    assert L.fb_fft1d_batched(p, p, 16, 0, None) == 1       # empty batch
    assert L.fb_ifft1d_batched(None, p, 16, 2, None) == 1
    assert L.fb_fft1d_batched(ctypes.c_void_p(8), p, 16, 2, None) == 3
    assert L.fb_fft1d_batched(p, ctypes.c_void_p((1 << 20) + 64), 16, 2, None) == 1  # partial overlap


def test_gemm_ex_validation(L):
    p = ctypes.c_void_p(1 << 20)
    ws = ctypes.c_void_p(1 << 30)
    big = 1 << 40
    assert L.fb_gemm(2, 0, 0, 4, 4, 4, 1.0, p, 4, p, 4, 0.0, p, 4, ws, big, None) == 1   # dtype
    assert L.fb_gemm(1, 2, 0, 4, 4, 4, 1.0, p, 4, p, 4, 0.0, p, 4, ws, big, None) == 1   # trans flag
    assert L.fb_gemm(1, 1, 0, 8, 4, 4, 1.0, p, 4, p, 4, 0.0, ctypes.c_void_p(1 << 24), 4, ws, big, None) == 1  # lda < m
    assert L.fb_gemm(0, 0, 0, 4, 4, 4, 1.0, p, 4, ctypes.c_void_p(1 << 22), 4, 0.0,
                     ctypes.c_void_p(1 << 24), 4, None, 0, None) == 4                       # FP32 workspace
    # transposes and alpha/beta need no temporaries: FP32 needs the fb_matmul split workspace,
    # FP64 none
    assert L.fb_gemm_workspace_bytes(0, 1, 1, 64, 64, 64) == L.fb_matmul_workspace_bytes(0, 64, 64, 64) > 0
    assert L.fb_gemm_workspace_bytes(1, 1, 1, 64, 64, 64) == 0


def test_rfft2d_validation(L):
    p = ctypes.c_void_p(1 << 20)
    q = ctypes.c_void_p(1 << 24)
    w = ctypes.c_void_p(1 << 28)
    assert L.fb_rfft2d(p, q, 4, 1, w, 1 << 20, None) == 1        # n1 < 2
    assert L.fb_rfft2d(p, q, 3, 8, w, 1 << 20, None) == 2        # not a power of two
    assert L.fb_rfft2d(p, q, 4, 8, None, 0, None) == 4           # workspace
    assert L.fb_irfft2d(p, ctypes.c_void_p((1 << 20) + 16), 4, 8, w, 1 << 20, None) == 1  # overlap
    assert L.fb_rfft2d_workspace_bytes(64, 64) >= 64 * 32 * 8 + 64 * 33 * 8
