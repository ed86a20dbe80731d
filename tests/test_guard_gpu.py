"""Out-of-bounds write checks for every entry point (a substitute for compute-sanitizer memcheck,
which this GPU pool does not allow: profiles/r2_sanitizer_closed.txt).

Every operand, result and workspace of a call is carved out of ONE device buffer, each followed
by a 4 KiB guard band; the whole buffer starts filled with the byte 0xA5.  After the call (and a
device synchronise) every guard byte must still be 0xA5 and every read-only operand must be
unchanged, so a kernel that writes past the end of any of its buffers, or into an input, fails
here.  Shapes are ragged against the kernels' tiles and cover each plan (cluster 256^2, pair
plan, four-step, the 16384-long row kernel, mixed radix, Bluestein, split + tcgen05 GEMM, DMMA,
BF16, BLAS-form transposes with alpha/beta, LU)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb():
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2004_09883_b200 as m
    torch.cuda.set_device(0)
    m.fb_init(0)
    return m


GUARD = 4096
CANARY = 0xA5


class Arena:
    def __init__(self, nbytes_list):
        self.offs, cur = [], GUARD
        for nb in nbytes_list:
            cur = (cur + 255) // 256 * 256
            self.offs.append(cur)
            cur += max(nb, 1) + GUARD
        self.sizes = [max(nb, 1) for nb in nbytes_list]
        self.buf = torch.full((cur + GUARD,), CANARY, dtype=torch.uint8, device="cuda")

    def view(self, i, dtype, shape):
        t = self.buf[self.offs[i]:self.offs[i] + self.sizes[i]]
        n = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
        return t[:n].view(dtype).view(*shape)

    def raw(self, i):
        return self.buf[self.offs[i]:self.offs[i] + self.sizes[i]]

    def guards_intact(self):
        torch.cuda.synchronize()
        mask = torch.ones_like(self.buf, dtype=torch.bool)
        for o, nb in zip(self.offs, self.sizes):
            mask[o:o + nb] = False
        return bool((self.buf[mask] == CANARY).all().item())


def _ptr(t):
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("n0,n1", [(256, 256), (2048, 2048), (8192, 256), (64, 16384), (1000, 360), (12, 8191),
                                   (512, 64), (16, 8)])
@pytest.mark.parametrize("inplace", [False, True])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft2d_guards(fb, n0, n1, inplace, inverse):
    L = fb.lib()
    nb = n0 * n1 * 8
    wsb = L.fb_fft2d_workspace_bytes(n0, n1)
    ar = Arena([nb, nb, wsb])
    x = ar.view(0, torch.complex64, (n0, n1))
    x.copy_(torch.from_numpy(synth.complex_field(n0, n1)).cuda())
    x0 = x.clone()
    y = x if inplace else ar.view(1, torch.complex64, (n0, n1))
    f = L.fb_ifft2d if inverse else L.fb_fft2d
    assert f(_ptr(x), _ptr(y), n0, n1, _ptr(ar.raw(2)), wsb, _stream()) == 0
    assert ar.guards_intact()
    if not inplace:
        assert torch.equal(x, x0)  # the input is read-only
        assert (ar.raw(1)[nb:] == CANARY).all()


@pytest.mark.parametrize("b,n", [(300, 16384), (37, 2048), (5, 64)])
def test_fft1d_guards(fb, b, n):
    L = fb.lib()
    nb = b * n * 8
    ar = Arena([nb, nb])
    x = ar.view(0, torch.complex64, (b, n))
    x.copy_(torch.from_numpy(synth.complex_field(b, n)).cuda())
    x0 = x.clone()
    y = ar.view(1, torch.complex64, (b, n))
    assert L.fb_fft1d_batched(_ptr(x), _ptr(y), n, b, _stream()) == 0
    assert ar.guards_intact() and torch.equal(x, x0)


@pytest.mark.parametrize("n0,n1", [(512, 256), (64, 2048), (2, 4)])
def test_rfft2d_guards(fb, n0, n1):
    L = fb.lib()
    h = n1 // 2 + 1
    wsb = L.fb_rfft2d_workspace_bytes(n0, n1)
    ar = Arena([n0 * n1 * 4, n0 * h * 8, wsb, n0 * n1 * 4])
    x = ar.view(0, torch.float32, (n0, n1))
    x.copy_(torch.from_numpy(np.ascontiguousarray(synth.real_matrix(n0, n1, synth.TID_NOISE))).cuda())
    x0 = x.clone()
    y = ar.view(1, torch.complex64, (n0, h))
    assert L.fb_rfft2d(_ptr(x), _ptr(y), n0, n1, _ptr(ar.raw(2)), wsb, _stream()) == 0
    y0 = y.clone()
    z = ar.view(3, torch.float32, (n0, n1))
    assert L.fb_irfft2d(_ptr(y), _ptr(z), n0, n1, _ptr(ar.raw(2)), wsb, _stream()) == 0
    assert ar.guards_intact() and torch.equal(x, x0) and torch.equal(y, y0)


@pytest.mark.parametrize("dt,m,n,k", [(torch.float32, 300, 264, 200), (torch.float32, 14400, 4700 // 4 * 4, 64),
                                      (torch.float32, 1, 4, 4), (torch.float64, 301, 262, 198),
                                      (torch.float64, 65, 2, 2)])
def test_matmul_guards(fb, dt, m, n, k):
    L = fb.lib()
    es = torch.empty(0, dtype=dt).element_size()
    code = fb.FB_F32 if dt == torch.float32 else fb.FB_F64
    wsb = L.fb_matmul_workspace_bytes(code, m, n, k)
    ar = Arena([m * k * es, k * n * es, m * n * es, wsb])
    A = ar.view(0, dt, (m, k))
    B = ar.view(1, dt, (k, n))
    A.copy_(torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(dt))
    B.copy_(torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(dt))
    A0, B0 = A.clone(), B.clone()
    C = ar.view(2, dt, (m, n))
    assert L.fb_matmul(code, m, n, k, _ptr(A), k, _ptr(B), n, _ptr(C), n, _ptr(ar.raw(3)) if wsb else None, wsb,
                       _stream()) == 0
    assert ar.guards_intact() and torch.equal(A, A0) and torch.equal(B, B0)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_gemm_guards(fb, dt, ta, tb):
    L = fb.lib()
    m, n, k = 300, 260, 204
    es = torch.empty(0, dtype=dt).element_size()
    code = fb.FB_F32 if dt == torch.float32 else fb.FB_F64
    wsb = L.fb_gemm_workspace_bytes(code, ta, tb, m, n, k)
    ar_shape_a = (k, m) if ta else (m, k)
    ar_shape_b = (n, k) if tb else (k, n)
    ar = Arena([m * k * es, k * n * es, m * n * es, wsb])
    A = ar.view(0, dt, ar_shape_a)
    B = ar.view(1, dt, ar_shape_b)
    C = ar.view(2, dt, (m, n))
    A.copy_(torch.from_numpy(synth.real_matrix(*ar_shape_a, synth.TID_GEMM_A)).to(dt))
    B.copy_(torch.from_numpy(synth.real_matrix(*ar_shape_b, synth.TID_GEMM_B)).to(dt))
    C.copy_(torch.from_numpy(synth.real_matrix(m, n, synth.TID_NOISE)).to(dt))
    A0, B0 = A.clone(), B.clone()
    assert L.fb_gemm(code, ta, tb, m, n, k, 0.75, _ptr(A), A.stride(0), _ptr(B), B.stride(0), -0.5, _ptr(C), n,
                     _ptr(ar.raw(3)) if wsb else None, wsb, _stream()) == 0
    assert ar.guards_intact() and torch.equal(A, A0) and torch.equal(B, B0)


@pytest.mark.parametrize("bt", [True, False])
def test_matmul_bf16_guards(fb, bt):
    L = fb.lib()
    m, n, k = 520, 392, 136
    wsb = L.fb_matmul_bf16_workspace_bytes(int(bt), m, n, k)
    shape_b = (n, k) if bt else (k, n)
    ar = Arena([m * k * 2, k * n * 2, m * n * 4, wsb])
    A = ar.view(0, torch.bfloat16, (m, k))
    B = ar.view(1, torch.bfloat16, shape_b)
    A.copy_(torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(torch.bfloat16))
    B.copy_(torch.from_numpy(synth.real_matrix(*shape_b, synth.TID_GEMM_B)).to(torch.bfloat16))
    A0, B0 = A.clone(), B.clone()
    C = ar.view(2, torch.float32, (m, n))
    assert L.fb_matmul_bf16(m, n, k, _ptr(A), k, _ptr(B), B.stride(0), int(bt), _ptr(C), n,
                            _ptr(ar.raw(3)) if wsb else None, wsb, _stream()) == 0
    assert ar.guards_intact() and torch.equal(A, A0) and torch.equal(B, B0)


@pytest.mark.parametrize("n", [300, 2048])
def test_lu_guards(fb, n):
    ar = Arena([n * n * 8, n * 4, 4])
    A = ar.view(0, torch.float64, (n, n))
    A.copy_(torch.from_numpy(synth.dct2_matrix(n)))
    ipiv = ar.view(1, torch.int32, (n,))
    info = ar.view(2, torch.int32, (1,))
    info.zero_()
    fb.fb_lu(A, ipiv, info)
    assert ar.guards_intact()
