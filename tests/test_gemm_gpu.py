"""GPU parity of the matrix block (fb_matmul through the C ABI) against the oracle.

Bars (north_star): FP64 rel-L2 <= 1e-12, FP32 (3xTF32) rel-L2 <= 1e-5.
"""
import numpy as np
import pytest
import torch

import oracle
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


def _mm(fb, A, B):
    C = fb.matmul(torch.from_numpy(np.ascontiguousarray(A)).cuda(), torch.from_numpy(np.ascontiguousarray(B)).cuda())
    torch.cuda.synchronize()
    return C.cpu().numpy()


SHAPES = [(1, 1, 1), (1, 4, 4), (4, 4, 1), (16, 16, 16), (128, 128, 32), (130, 132, 36), (255, 260, 300),
          (511, 384, 257), (1000, 40, 1030), (64, 1024, 8), (300, 300, 4)]


def _mm_padded(fb, A, B):
    """A (m x k) and B (k x n) in buffers whose rows are padded to 16 bytes (the C-ABI rule
    ld*elemsize % 16 == 0), passed as strided views; C likewise.  Ragged k and n then run."""
    es = A.itemsize
    q = 16 // es
    m, k = A.shape
    n = B.shape[1]
    dt = torch.float32 if es == 4 else torch.float64
    Ab = torch.zeros(m, -(-k // q) * q, dtype=dt)
    Bb = torch.zeros(k, -(-n // q) * q, dtype=dt)
    Ab[:, :k] = torch.from_numpy(A)
    Bb[:, :n] = torch.from_numpy(B)
    Ab, Bb = Ab.cuda(), Bb.cuda()
    Cb = torch.full((m, Bb.shape[1]), 7.0, dtype=dt, device="cuda")
    fb.matmul(Ab[:, :k], Bb[:, :n], out=Cb[:, :n])
    torch.cuda.synchronize()
    assert torch.all(Cb[:, n:] == 7.0)  # padding columns of C untouched
    return Cb[:, :n].cpu().numpy()


@pytest.mark.parametrize("m,n,k", SHAPES)
def test_f64_ragged_vs_oracle(fb, m, n, k):
    A = synth.real_matrix(m, k, synth.TID_GEMM_A, dtype=np.float64)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B, dtype=np.float64)
    assert oracle.rel_l2(_mm_padded(fb, A, B), oracle.matmul(A, B)) < 1e-12


@pytest.mark.parametrize("m,n,k", SHAPES)
def test_f32_ragged_vs_oracle(fb, m, n, k):
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    assert oracle.rel_l2(_mm_padded(fb, A, B), oracle.matmul(A, B)) < 1e-5


@pytest.mark.parametrize("m,n,k", [(255, 260, 300), (2048, 2048, 2048), (130, 132, 36)])
def test_f64_full_mantissa_vs_oracle(fb, m, n, k):
    """Full 53-bit-mantissa inputs: every product rounds, so the 1e-12 bar probes the DMMA
    products and the accumulation, not only the summation order (24-bit inputs multiply exactly)."""
    A = synth.real_matrix_f64(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix_f64(k, n, synth.TID_GEMM_B)
    err = oracle.rel_l2(_mm(fb, A, B), oracle.matmul(A, B))
    assert err < 1e-12, err


def test_f32_padded_leading_dims(fb):
    m, n, k = 200, 100, 150
    Ab = torch.from_numpy(synth.real_matrix(m, 160, synth.TID_GEMM_A)).cuda()
    Bb = torch.from_numpy(synth.real_matrix(k, 128, synth.TID_GEMM_B)).cuda()
    A, B = Ab[:, :k], Bb[:, :n]
    Cb = torch.zeros(m, 104, device="cuda")
    fb.matmul(A, B, out=Cb[:, :n])
    torch.cuda.synchronize()
    ref = oracle.matmul(A.cpu().numpy().copy(), B.cpu().numpy().copy())
    assert oracle.rel_l2(Cb[:, :n].cpu().numpy(), ref) < 1e-5
    assert torch.all(Cb[:, n:] == 0)


@pytest.mark.parametrize("m,n,k", [(200, 100, 150), (300, 260, 203), (2048, 2048, 2048), (64, 1000, 8)])
def test_f32_wide_split_bitwise(fb, m, n, k, monkeypatch):
    """The wide operand split (split_both_wide_kernel: flattened float4 chunks of A, 64 x 64
    tiles of B, ragged k and n) with RNA hi/lo for A (FB_GEMM_AHI_RAW=0) gives C bit for bit equal
    to the 32 x 32-tile split_both_kernel (knob FB_GEMM_SPLITV=1): same split per element, same
    GEMM.  The default (raw A as the hi operand, only lo = rna(a - trunc(a)) written; reading R21)
    is a different decomposition: within the bar and bitwise deterministic."""
    Ab = torch.from_numpy(synth.real_matrix(m, (k + 3) // 4 * 4, synth.TID_GEMM_A)).cuda()
    Bb = torch.from_numpy(synth.real_matrix(k, (n + 3) // 4 * 4, synth.TID_GEMM_B)).cuda()
    A, B = Ab[:, :k], Bb[:, :n]
    C2 = fb.matmul(A, B)
    C3 = fb.matmul(A, B)
    monkeypatch.setenv("FB_GEMM_AHI_RAW", "0")
    C1 = fb.matmul(A, B)
    torch.cuda.synchronize()
    monkeypatch.setenv("FB_GEMM_SPLITV", "1")
    C0 = fb.matmul(A, B)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1) and torch.equal(C2, C3)
    if m * n * k <= 2 ** 24:
        ref = oracle.matmul(A.cpu().numpy().copy(), B.cpu().numpy().copy())
        assert oracle.rel_l2(C1.cpu().numpy(), ref) < 1e-5
        assert oracle.rel_l2(C2.cpu().numpy(), ref) < 1e-5


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_2048_config2_full_oracle(fb, dt):
    """BASELINE configs[2]: 2048^3 in FP64 and FP32, full oracle."""
    n = 2048
    A = synth.real_matrix(n, n, synth.TID_GEMM_A, dtype=dt)
    B = synth.real_matrix(n, n, synth.TID_GEMM_B, dtype=dt)
    err = oracle.rel_l2(_mm(fb, A, B), oracle.matmul(A, B))
    assert err < (1e-5 if dt == np.float32 else 1e-12), err


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_identity_permutation_hadamard(fb, dt):
    n = 512
    A = synth.real_matrix(n, n, synth.TID_GEMM_A, dtype=dt)
    I = np.eye(n, dtype=dt)
    if dt == np.float64:
        assert np.array_equal(_mm(fb, A, I), A)  # exact in FP64
    else:
        # 3xTF32: A*I = hi + lo (+ lo*hi term 0) -> within 1 ulp elementwise
        assert np.abs(_mm(fb, A, I) - A).max() <= np.abs(A).max() * 2 ** -22
    p = np.random.default_rng(1).permutation(n)
    P = np.eye(n, dtype=dt)[p]
    got = _mm(fb, P, A)
    assert np.abs(got - A[p]).max() <= (0 if dt == np.float64 else np.abs(A).max() * 2 ** -22)
    H = synth.hadamard(n).astype(dt)
    assert np.array_equal(_mm(fb, H, np.ascontiguousarray(H.T)), n * np.eye(n, dtype=dt))


def test_dct_orthogonal_f64(fb):
    """P:153 'orthogonal matrix data': Q Q^T = I for the orthonormal DCT-II."""
    Q = synth.dct2_matrix(2048)
    Qt = np.ascontiguousarray(Q.T)
    R = _mm(fb, Q, Qt)
    # Q itself is FP64-rounded: even the exact product of the stored Q deviates from I by
    # ~1.05e-13 (numpy and the oracle agree), so the bar is 2e-13 plus oracle parity.
    assert np.abs(R - np.eye(2048)).max() < 2e-13
    assert oracle.rel_l2(R, oracle.matmul(Q, Qt)) < 1e-12


def test_deterministic(fb):
    A = synth.real_matrix(1024, 1024, synth.TID_GEMM_A)
    B = synth.real_matrix(1024, 1024, synth.TID_GEMM_B)
    assert np.array_equal(_mm(fb, A, B), _mm(fb, A, B))


def test_tc_operand_truncation_probe(fb):
    """Reading R21 pin (the raw-A-hi default depends on it): fed a raw FP32 operand
    x = 1 + 2^-11 + 2^-12 (not TF32-exact; round-to-nearest gives 1 + 2^-10, truncation 1.0),
    kind::tf32 multiplies trunc(x): C = sum over k = 8 of hi(x) * 1 = 8 exactly, never 8 + 2^-7."""
    m = n = 128
    k = 8
    x = np.float32(1 + 2.0 ** -11 + 2.0 ** -12)
    Ah = torch.full((m, k), float(x), device="cuda")
    Al = torch.zeros(m, k, device="cuda")
    Bh = torch.ones(n, k, device="cuda")
    Bl = torch.zeros(n, k, device="cuda")
    C = torch.empty(m, n, device="cuda")
    fb.fb_matmul_3xtf32_presplit(Ah, Al, Bh, Bl, C)
    torch.cuda.synchronize()
    assert torch.all(C == 8.0), float(C[0, 0])
    # and the full path keeps x exactly through hi = trunc(x), lo = rna(x - trunc(x))
    A = torch.full((m, k), float(x), device="cuda")
    Cm = fb.matmul(A, torch.ones(k, n, device="cuda"))
    torch.cuda.synchronize()
    assert torch.all(Cm == float(8 * np.float64(x))), float(Cm[0, 0])


def test_tc_accumulation_rounding_probe(fb):
    """Reading R11 probe: one k-block adds 0.75 ulp(1) to an accumulator holding 1.0.
    RN accumulation gives 1 + 2^-23, RZ gives 1.0.  Recorded, and the K=32768 test below
    decides whether the 3xTF32 path meets 1e-5 either way."""
    k = 64
    A = np.zeros((128, k), np.float32)
    B = np.zeros((k, 128), np.float32)
    A[0, 0] = 1.0
    B[0, 0] = 1.0
    A[0, 40] = 0.75 * 2 ** -23   # TF32-exact, second k-block (BK = 32)
    B[40, 0] = 1.0
    c = _mm(fb, A, B)[0, 0]
    mode = "RN" if c == np.float32(1 + 2 ** -23) else ("RZ" if c == 1.0 else f"other({c!r})")
    print(f"tcgen05 FP32 accumulation behaves as {mode}")
    assert mode in ("RN", "RZ")


def test_f32_k32768_sampled(fb):
    """Long-K accuracy (configs[4] K): rows sampled vs the oracle."""
    m, n, k = 256, 256, 32768
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    C = _mm(fb, A, B)
    rows = [0, 1, 128, 255]
    err = oracle.rel_l2(C[rows], oracle.matmul_rows(A, B, rows))
    print(f"K=32768 3xTF32 rel-L2 {err:.3e}")
    assert err < 1e-5


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_large_sampled_rows(fb, dt):
    """4096^3 (FP32: 256 x 240 pair tiles in 4 waves; FP64: 4096 DMMA tiles) with full-mantissa
    FP64 inputs where applicable: sampled full rows, including the first and last, against the
    oracle's row function."""
    n = 4096
    mk = synth.real_matrix_f64 if dt == torch.float64 else synth.real_matrix
    A, B = mk(n, n, synth.TID_GEMM_A), mk(n, n, synth.TID_GEMM_B)
    C = _mm(fb, A, B)
    rows = [0, 1, 255, 256, 2047, 4095]
    err = oracle.rel_l2(C[rows], oracle.matmul_rows(A, B, rows))
    assert err < (1e-5 if dt == torch.float32 else 1e-12), err


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_gemm_ex_transposed_large(fb, dt):
    """fb_gemm with both operands transposed and alpha/beta at 2048^3 (FP32 picks 256 x 240
    tiles): sampled rows against alpha op(A) op(B) + beta C0 formed by the oracle in FP64."""
    n = 2048
    mk = synth.real_matrix_f64 if dt == torch.float64 else synth.real_matrix
    At, Bt, C0 = mk(n, n, synth.TID_GEMM_A), mk(n, n, synth.TID_GEMM_B), mk(n, n, synth.TID_NOISE)
    C = torch.from_numpy(C0).to(dt).cuda()
    fb.gemm(torch.from_numpy(At).to(dt).cuda(), torch.from_numpy(Bt).to(dt).cuda(), C, 1.5, -0.25, True, True)
    torch.cuda.synchronize()
    rows = [0, 777, 2047]
    opA = np.ascontiguousarray(At.T).astype(np.float64)
    opB = np.ascontiguousarray(Bt.T).astype(np.float64)
    ref = 1.5 * oracle.matmul_rows(opA, opB, rows) - 0.25 * C0[rows].astype(np.float64)
    err = oracle.rel_l2(C.cpu().numpy()[rows], ref)
    assert err < (1e-5 if dt == torch.float32 else 1e-12), err


def test_host_variant(fb):
    m, n, k = 300, 256, 128
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).pin_memory()
    B = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).pin_memory()
    C = torch.empty(m, n).pin_memory()
    fb.fb_matmul_host(A, B, C)
    assert oracle.rel_l2(C.numpy(), oracle.matmul(A.numpy(), B.numpy())) < 1e-5


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_gemm_ex_transposes_alpha_beta(fb, dt, ta, tb):
    """fb_gemm: C = alpha op(A) op(B) + beta C against the oracle product of the
    explicitly transposed operands, combined with alpha, beta in FP64."""
    m, n, k = 200, 136, 72
    Ah = synth.real_matrix(k if ta else m, m if ta else k, synth.TID_GEMM_A)
    Bh = synth.real_matrix(n if tb else k, k if tb else n, synth.TID_GEMM_B)
    C0 = synth.real_matrix(m, n, synth.TID_NOISE)
    opA = Ah.T if ta else Ah
    opB = Bh.T if tb else Bh
    P = oracle.matmul(np.ascontiguousarray(opA).astype(np.float64), np.ascontiguousarray(opB).astype(np.float64))
    bar = 1e-5 if dt == torch.float32 else 1e-12
    for alpha, beta in [(1.0, 0.0), (0.75, -0.5), (-2.0, 1.0)]:
        A = torch.from_numpy(np.ascontiguousarray(Ah)).to(dt).cuda()
        B = torch.from_numpy(np.ascontiguousarray(Bh)).to(dt).cuda()
        C = torch.from_numpy(C0).to(dt).cuda()
        fb.gemm(A, B, C, alpha, beta, bool(ta), bool(tb))
        torch.cuda.synchronize()
        ref = alpha * P + beta * C0.astype(np.float64)
        assert oracle.rel_l2(C.cpu().numpy(), ref) < bar, (alpha, beta)


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("ta,tb", [(1, 0), (0, 1), (1, 1)])
def test_gemm_ex_transposed_operand_bitwise(fb, dt, ta, tb):
    """A transposed operand is read in its stored orientation (FP64 tile loads, FP32 TF32
    split), so fb_gemm(trans) is bitwise fb_matmul on the explicitly transposed operands (same
    values, same k order), across several tiles with ragged edges; (alpha, beta) = (1, 0)."""
    m, n, k = 300, 260, 203
    mk = synth.real_matrix_f64 if dt == torch.float64 else synth.real_matrix
    Ah = mk(k if ta else m, m if ta else k, synth.TID_GEMM_A)
    Bh = mk(n if tb else k, k if tb else n, synth.TID_GEMM_B)
    opA = np.ascontiguousarray(Ah.T if ta else Ah)
    opB = np.ascontiguousarray(Bh.T if tb else Bh)
    q = 16 // np.dtype(np.float64 if dt == torch.float64 else np.float32).itemsize

    def dev(h):  # 16-byte row pitch as the ABI requires
        b = torch.zeros(h.shape[0], -(-h.shape[1] // q) * q, dtype=dt)
        b[:, :h.shape[1]] = torch.from_numpy(np.ascontiguousarray(h)).to(dt)
        return b.cuda()[:, :h.shape[1]]

    C1 = dev(np.zeros((m, n)))
    fb.gemm(dev(Ah), dev(Bh), C1, 1.0, 0.0, bool(ta), bool(tb))
    C0 = dev(np.zeros((m, n)))
    fb.gemm(dev(opA), dev(opB), C0, 1.0, 0.0)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1)
    bar = 1e-5 if dt == torch.float32 else 1e-12
    assert oracle.rel_l2(C1.cpu().numpy(), oracle.matmul(opA.astype(np.float64), opB.astype(np.float64))) < bar


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_gemm_ex_epilogue_large(fb, dt):
    """alpha/beta in the epilogue over many tiles (FP32 pair kernel 256 x 256 tiles, FP64 64 x 64),
    full-mantissa FP64 operands, against alpha P + beta C0 formed in FP64 by the oracle."""
    m, n, k = 700, 532, 332  # ld*4 % 16 == 0 (ABI), ragged against the 256 and 64 tiles
    mk = synth.real_matrix_f64 if dt == torch.float64 else synth.real_matrix
    A0, B0, C0 = mk(m, k, synth.TID_GEMM_A), mk(k, n, synth.TID_GEMM_B), mk(m, n, synth.TID_NOISE)
    P = oracle.matmul(A0.astype(np.float64), B0.astype(np.float64))
    for alpha, beta in [(0.75, -0.5), (1.0, 1.0), (-3.0, 0.0)]:
        C = torch.from_numpy(C0).to(dt).cuda()
        fb.gemm(torch.from_numpy(A0).to(dt).cuda(), torch.from_numpy(B0).to(dt).cuda(), C, alpha, beta)
        torch.cuda.synchronize()
        ref = alpha * P + beta * C0.astype(np.float64)
        assert oracle.rel_l2(C.cpu().numpy(), ref) < (1e-5 if dt == torch.float32 else 1e-12), (alpha, beta)


@pytest.mark.parametrize("ta,tb,m,n,k", [(1, 0, 128, 128, 6), (1, 1, 96, 40, 13), (0, 0, 100, 130, 64),
                                         (0, 1, 64, 130, 50), (1, 0, 33, 131, 7)])
def test_gemm_ex_f32_unaligned_temporaries(fb, ta, tb, m, n, k):
    """fb_gemm FP32 with k % 4 != 0 under transA and n % 4 != 0, n >= 128 with (alpha, beta) !=
    (1, 0): every operand and C live in 16-byte-pitched buffers, as the ABI requires, and the
    split / epilogue handle the ragged rows."""
    q = 4
    def padded(rows, cols, tid):
        h = synth.real_matrix(rows, cols, tid)
        b = torch.zeros(rows, -(-cols // q) * q)
        b[:, :cols] = torch.from_numpy(h)
        return h, b.cuda()[:, :cols]
    Ah, A = padded(k if ta else m, m if ta else k, synth.TID_GEMM_A)
    Bh, B = padded(n if tb else k, k if tb else n, synth.TID_GEMM_B)
    C0h, C = padded(m, n, synth.TID_NOISE)
    opA = Ah.T if ta else Ah
    opB = Bh.T if tb else Bh
    P = oracle.matmul(np.ascontiguousarray(opA).astype(np.float64), np.ascontiguousarray(opB).astype(np.float64))
    alpha, beta = 0.75, -0.5
    fb.gemm(A, B, C, alpha, beta, bool(ta), bool(tb))
    torch.cuda.synchronize()
    assert oracle.rel_l2(C.cpu().numpy(), alpha * P + beta * C0h.astype(np.float64)) < 1e-5


def test_gemm_ex_beta0_ignores_nan_and_alpha0(fb):
    m, n, k = 64, 48, 40
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).double().cuda()
    B = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).double().cuda()
    C = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    fb.gemm(A, B, C, 1.5, 0.0)
    ref = 1.5 * oracle.matmul(A.cpu().numpy(), B.cpu().numpy())
    torch.cuda.synchronize()
    assert torch.isfinite(C).all() and oracle.rel_l2(C.cpu().numpy(), ref) < 1e-12
    C2 = torch.ones(m, n, dtype=torch.float64, device="cuda")
    fb.gemm(A, B, C2, 0.0, 3.0)
    torch.cuda.synchronize()
    assert torch.equal(C2, torch.full_like(C2, 3.0))


@pytest.mark.parametrize("knobs,dt", [({"FB_GEMM_1CTA": "1"}, torch.float32), ({"FB_GEMM_SPLIT2": "1"}, torch.float32),
                                      ({"FB_GEMM_SPLITV": "1"}, torch.float32),
                                      ({"FB_F64_CFG": "1"}, torch.float64), ({"FB_F64_CFG": "2"}, torch.float64)])
def test_gemm_path_variants(fb, knobs, dt, monkeypatch):
    """The kernels behind A/B knobs (1-CTA tcgen05 kernel, two split launches, the larger FP64
    tile shapes) match the oracle like the defaults."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    m, n, k = 320, 264, 200
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(dt).cuda()
    B = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(dt).cuda()
    C = fb.matmul(A, B)
    torch.cuda.synchronize()
    bar = 1e-5 if dt == torch.float32 else 1e-12
    assert oracle.rel_l2(C.cpu().numpy(), oracle.matmul(A.cpu().numpy(), B.cpu().numpy())) < bar


@pytest.mark.parametrize("knobs", [{"FB_GEMM_FUSED": "1"}, {"FB_GEMM_FUSED": "1", "FB_GEMM_STREAMK": "1"},
                                   {"FB_GEMM_FUSED": "1", "FB_GEMM_LO_OVERLAP": "1"},
                                   {"FB_GEMM_FUSED": "1", "FB_GEMM_LO_PREPASS": "0"}])
@pytest.mark.parametrize("m,n,k", [(300, 260, 203), (2048, 2048, 2048), (2048, 2048, 512), (64, 1000, 8), (1, 1, 1)])
def test_gemm_fused_kernel_vs_oracle(fb, knobs, m, n, k, monkeypatch):
    """The single-kernel FP32 path (fb_gemm_fused.cu: raw operands as the truncated TF32 hi part,
    lo from a streaming pre-pass or formed in shared memory, B consumed MN-major, stream-K over
    all SM pairs with a deterministic fix-up) against the oracle, and bitwise run to run."""
    for kk, v in knobs.items():
        monkeypatch.setenv(kk, v)
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    C1 = _mm_padded(fb, A, B)
    C2 = _mm_padded(fb, A, B)
    assert np.array_equal(C1, C2)
    assert oracle.rel_l2(C1, oracle.matmul(A, B)) < 1e-5


@pytest.mark.parametrize("m,n,k", [(4096, 3000, 300), (2600, 2048, 1000), (300, 260, 203)])
def test_gemm_persistent_pair_bitwise(fb, m, n, k, monkeypatch):
    """FB_GEMM_PERSIST=1: 74 CTA pairs loop over the tiles (stage ring and TMEM accumulators
    running on across tiles).  Per tile the arithmetic is the non-persistent kernel's, so the
    result is bitwise the same, with more tiles than pairs and a ragged edge."""
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    C0 = _mm_padded(fb, A, B)
    monkeypatch.setenv("FB_GEMM_PERSIST", "1")
    C1 = _mm_padded(fb, A, B)
    assert np.array_equal(C0, C1)
    assert oracle.rel_l2(C1, oracle.matmul(A, B)) < 1e-5


@pytest.mark.parametrize("m,n,k", [(2048, 2048, 512), (600, 1000, 300), (300, 250, 64), (512, 4096, 136)])
def test_gemm_pair_tile_240_bitwise(fb, m, n, k, monkeypatch):
    """FB_GEMM_NT=240: CTA-pair tiles 256 x 240 (MMA N = 240, each CTA stages 120 rows of B^T,
    the epilogue drains 120 columns as 3 x32 + x16 + x8 TMEM loads).  A tile boundary does not
    change any element's arithmetic, so the product is bitwise the 256-wide tiles' one (auto
    picks 240 where it needs fewer waves x width, e.g. 2048^2)."""
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    monkeypatch.setenv("FB_GEMM_NT", "256")
    C0 = _mm_padded(fb, A, B)
    monkeypatch.setenv("FB_GEMM_NT", "240")
    C1 = _mm_padded(fb, A, B)
    assert np.array_equal(C0, C1)
    assert oracle.rel_l2(C1, oracle.matmul(A, B)) < 1e-5


@pytest.mark.parametrize("panel", ["0", "1024", "2048", "-1"])
def test_gemm_n_panels_bitwise(fb, panel, monkeypatch):
    """FP32 GEMM issued as N-column panel launches (auto for tall A: m >= ~14100; FB_GEMM_NPANEL
    forces a width) computes every element with the same arithmetic: bitwise equal to the
    single launch, ragged last panel included, and alpha/beta (fb_gemm) per panel."""
    m, n, k = 14400, 4700, 200  # auto: 57 tile rows -> panels of 2048 columns
    A = synth.real_matrix(m, k, synth.TID_GEMM_A)
    B = synth.real_matrix(k, n, synth.TID_GEMM_B)
    monkeypatch.setenv("FB_GEMM_NPANEL", "0")
    C0 = _mm_padded(fb, A, B)
    monkeypatch.setenv("FB_GEMM_NPANEL", panel)
    C1 = _mm_padded(fb, A, B)
    assert np.array_equal(C0, C1)
    rows = [0, 7777, m - 1]
    ref = oracle.matmul(A[rows].astype(np.float64), B.astype(np.float64))
    assert oracle.rel_l2(C1[rows], ref) < 1e-5
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B[:, :4696]).contiguous().cuda()
    Cd = torch.ones(m, 4696, device="cuda")
    fb.gemm(Ad, Bd, Cd, 0.5, -1.0)
    torch.cuda.synchronize()
    P = torch.from_numpy(C0[:, :4696]).cuda()
    assert torch.allclose(Cd, 0.5 * P - 1.0, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("m,n,k,bt", [(256, 256, 64, True), (300, 200, 136, False), (512, 768, 1000, True),
                                      (2048, 2048, 2048, False), (40, 24, 8, True)])
def test_gemm_bf16_vs_oracle(fb, m, n, k, bt):
    """fb_matmul_bf16: the product of the bf16 inputs (exact in FP64) within 1e-5
    (FP32 accumulation, RN promotion every 1024 k)."""
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(torch.bfloat16).cuda()
    Bk = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(torch.bfloat16).cuda()
    B = Bk.t().contiguous() if bt else Bk
    C = fb.matmul_bf16(A, B, b_transposed=bt)
    torch.cuda.synchronize()
    ref = oracle.matmul(A.float().cpu().numpy().astype(np.float64), Bk.float().cpu().numpy().astype(np.float64))
    assert oracle.rel_l2(C.cpu().numpy(), ref) < 1e-5


def test_gemm_bf16_k8192_sampled(fb):
    """Long K (8192 = 8 promotion intervals): sampled full rows against the exact product."""
    m, n, k = 512, 768, 8192
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(torch.bfloat16).cuda()
    Bk = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(torch.bfloat16).cuda()
    C = fb.matmul_bf16(A, Bk.t().contiguous(), b_transposed=True)
    torch.cuda.synchronize()
    rows = np.array([0, 1, 127, 128, 255, 300, 511])
    Ad = A.float().cpu().numpy().astype(np.float64)[rows]
    ref = oracle.matmul(Ad, Bk.float().cpu().numpy().astype(np.float64))
    assert oracle.rel_l2(C.cpu().numpy()[rows], ref) < 1e-5


def test_gemm_bf16_multicast_cluster(fb, monkeypatch):
    """The 4-CTA cluster variant (A tiles multicast to two CTA pairs) gives the same product
    bit for bit (same MMA order per tile), including an odd tile count along N."""
    m, n, k = 512, 768, 640
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(torch.bfloat16).cuda()
    Bt = torch.from_numpy(synth.real_matrix(n, k, synth.TID_GEMM_B)).to(torch.bfloat16).cuda()
    C2 = fb.matmul_bf16(A, Bt, b_transposed=True)
    monkeypatch.setenv("FB_BF16_CLUSTER", "4")
    C4 = fb.matmul_bf16(A, Bt, b_transposed=True)
    torch.cuda.synchronize()
    assert torch.equal(C2, C4)


def test_gemm_bf16_persistent_bitwise(fb, monkeypatch):
    """Persistent BF16 kernel (default): one CTA pair per 2 SMs loops over the tiles with the
    stage ring and TMEM accumulators running on across tiles; per tile the MMA order is
    unchanged, so the product is bitwise the one-tile-per-pair kernel's (FB_BF16_PERSIST=0),
    with more tiles than pairs and ragged edges."""
    m, n, k = 3000, 2900, 640
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(torch.bfloat16).cuda()
    Bt = torch.from_numpy(synth.real_matrix(n, k, synth.TID_GEMM_B)).to(torch.bfloat16).cuda()
    C1 = fb.matmul_bf16(A, Bt, b_transposed=True)
    monkeypatch.setenv("FB_BF16_PERSIST", "0")
    C0 = fb.matmul_bf16(A, Bt, b_transposed=True)
    torch.cuda.synchronize()
    assert torch.equal(C0, C1)


def test_config4_full_size_sampled(fb):
    """configs[4] at its full size (32768^3 FP32, the launch configuration bench.py times at one
    GPU): sampled full rows and columns of C against the oracle (each 2^30 FP64 MACs)."""
    n = 32768
    g = torch.Generator(device="cuda").manual_seed(200409883)
    A = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    B = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
    C = fb.matmul(A, B)
    torch.cuda.synchronize()
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    rows, cols = [0, 12345, n - 1], [0, 777, n - 1]
    Ch = C.cpu().numpy()
    del A, B, C
    torch.cuda.empty_cache()
    err_r = oracle.rel_l2(Ch[rows], oracle.matmul_rows(Ah, Bh, rows))
    err_c = oracle.rel_l2(Ch[:, cols].T, oracle.matmul_cols(Ah, Bh, cols))
    print(f"32768^3 3xTF32 sampled rel-L2 rows {err_r:.3e} cols {err_c:.3e}")
    assert err_r < 1e-5 and err_c < 1e-5
