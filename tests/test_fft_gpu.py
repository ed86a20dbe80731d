"""GPU parity of the Fourier block (fb_fft2d / fb_ifft2d through the C ABI) against the oracle.

Bars (north_star): rel-L2 <= 1e-5 * log2(n0 n1); internal gate 5e-7 on uniform inputs
(reading R6) for sizes where the full oracle runs.
"""
import itertools

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


def _bar(n0, n1):
    return 1e-5 * max(1.0, np.log2(n0 * n1))


def _run(fb, x, inverse=False, inplace=False):
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if inplace:
        fb.fft2d(xd, out=xd, inverse=inverse)
        out = xd
    else:
        out = fb.fft2d(xd, inverse=inverse)
    torch.cuda.synchronize()
    return out.cpu().numpy()


SMALL = [1, 2, 4, 8, 16, 32, 64, 128]


@pytest.mark.parametrize("n0,n1", list(itertools.product(SMALL, SMALL)))
def test_small_all_shapes_vs_oracle(fb, n0, n1):
    x = synth.complex_field(n0, n1, tensor_id=n0 * 1000 + n1)
    for inv in (False, True):
        y = _run(fb, x, inverse=inv)
        ref = oracle.dft2d(x, inverse=inv)
        err = oracle.rel_l2(y, ref)
        assert err < min(_bar(n0, n1), 5e-7), (n0, n1, inv, err)


@pytest.mark.parametrize("n0,n1", [(256, 256), (512, 256), (256, 1024), (1024, 64), (64, 2048)])
def test_full_oracle(fb, n0, n1):
    x = synth.complex_field(n0, n1)
    ref = oracle.dft2d(x)
    y = _run(fb, x)
    assert oracle.rel_l2(y, ref) < 5e-7
    z = _run(fb, y.astype(np.complex64), inverse=True)
    assert oracle.rel_l2(z, oracle.dft2d(y.astype(np.complex64), inverse=True)) < 5e-7


@pytest.mark.parametrize("small", ["8", "16", "0"])
def test_fft256_cluster_kernel_vs_oracle(fb, small, monkeypatch):
    """configs[0] as one thread-block-cluster kernel (fb_fft_small.cu; FB_FFT_SMALL = cluster size
    8 or 16, 0 = the two-pass path): forward against the full oracle, inverse round trip, in place
    (x == y), bitwise deterministic, and a single tone lands in one bin."""
    monkeypatch.setenv("FB_FFT_SMALL", small)
    xh = synth.complex_field(256, 256)
    x = torch.from_numpy(xh).cuda()
    y = fb.fft2d(x)
    y2 = fb.fft2d(x)
    z = fb.fft2d(y, inverse=True)
    w = x.clone()
    fb.fft2d(w, out=w)
    torch.cuda.synchronize()
    assert torch.equal(y, y2) and torch.equal(w, y)
    assert oracle.rel_l2(y.cpu().numpy(), oracle.dft2d(xh)) < 5e-7
    assert oracle.rel_l2(z.cpu().numpy(), xh) < 5e-7
    i0, i1 = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    tone = np.exp(2j * np.pi * (3 * i0 + 250 * i1) / 256).astype(np.complex64)
    yt = fb.fft2d(torch.from_numpy(tone).cuda()).cpu().numpy()
    ref = np.zeros((256, 256), np.complex128)
    ref[3, 250] = 65536
    assert np.abs(yt - ref).max() < 65536 * 1e-5


def test_256_forward_inverse_config0(fb):
    """BASELINE configs[0]: 256x256 fp32, single forward + inverse."""
    x = synth.complex_field(256, 256)
    y = _run(fb, x)
    assert oracle.rel_l2(y, oracle.dft2d(x)) < 5e-7
    z = _run(fb, y, inverse=True)
    assert oracle.rel_l2(z, x) < 5e-7


def test_inplace_equals_out_of_place(fb):
    x = synth.complex_field(512, 512)
    a = _run(fb, x)
    b = _run(fb, x, inplace=True)
    assert np.array_equal(a, b)


def test_deterministic(fb):
    x = synth.complex_field(1024, 1024)
    assert np.array_equal(_run(fb, x), _run(fb, x))


def _sampled_check(fb, n0, n1, x, y, ks0, ks1, inverse=False, tol=5e-7):
    for k1 in ks1:
        ref = oracle.dft2d_col(x, k1, inverse=inverse)
        e = oracle.rel_l2(y[:, k1], ref)
        assert e < tol, ("col", k1, e)
    for k0 in ks0:
        ref = oracle.dft2d_row(x, k0, inverse=inverse)
        e = oracle.rel_l2(y[k0, :], ref)
        assert e < tol, ("row", k0, e)


def test_2048_config1_sampled_and_closed_forms(fb):
    """BASELINE configs[1]: 2048x2048 -- sampled full rows/columns vs the oracle, plus
    Parseval and roundtrip at full size."""
    n = 2048
    x = synth.complex_field(n, n)
    y = _run(fb, x)
    _sampled_check(fb, n, n, x, y, [0, 1, 1023, 2047], [0, 5, 1024, 2047])
    xs = x.astype(np.complex128)
    assert np.isclose(np.sum(np.abs(y.astype(np.complex128)) ** 2), n * n * np.sum(np.abs(xs) ** 2), rtol=1e-5)
    z = _run(fb, y, inverse=True)
    assert oracle.rel_l2(z, x) < 5e-7


def test_2048_config1_full_oracle_fwd_inv(fb):
    """BASELINE configs[1] at its full size against the FULL oracle (every output element), in
    the launch configuration bench.py times: forward, and inverse of the forward's output."""
    n = 2048
    x = synth.complex_field(n, n)
    y = _run(fb, x)
    e_fwd = oracle.rel_l2(y, oracle.dft2d(x))
    z = _run(fb, y, inverse=True)
    e_inv = oracle.rel_l2(z, oracle.dft2d(y, inverse=True))
    print(f"2048^2 full oracle: forward {e_fwd:.3e} inverse {e_inv:.3e}")
    assert e_fwd < 5e-7 and e_inv < 5e-7


def test_2048_tones(fb):
    """Paper-shaped input (P:149 vibration analysis): integer tones + noise; the spectrum
    peaks sit exactly at the tone frequencies."""
    n = 2048
    x, tones = synth.tones2d(n, n)
    y = _run(fb, x)
    mag = np.abs(y)
    top = set(zip(*np.unravel_index(np.argsort(mag.ravel())[-len(tones):], mag.shape)))
    assert {(f0, f1) for f0, f1, _ in tones} == {(int(a), int(b)) for a, b in top}
    for k1 in sorted({f1 for _, f1, _ in tones})[:3]:
        assert oracle.rel_l2(y[:, k1], oracle.dft2d_col(x, k1)) < 1e-5


@pytest.mark.parametrize("n0,n1", [(8192, 64), (16384, 32), (8192, 256)])
def test_four_step_columns(fb, n0, n1):
    x = synth.complex_field(n0, n1)
    y = _run(fb, x)
    _sampled_check(fb, n0, n1, x, y, [0, 3, n0 - 1], [0, 7, n1 - 1])
    z = _run(fb, y, inverse=True)
    assert oracle.rel_l2(z, x) < 5e-7


def test_16384_square_sampled(fb):
    """configs[3] size on one GPU: 16384 x 16384 (2 GiB): 16 full output rows and 16 full output
    columns against the oracle -- the first and last line of every slab at P = 8 (which include
    those of P = 2 and 4), for both the row slabs and the column slabs -- plus the tone closed form."""
    n = 16384
    x = synth.complex_field(n, n)
    y = _run(fb, x)
    edges = sorted({b for r in range(8) for b in (r * n // 8, (r + 1) * n // 8 - 1)})
    assert len(edges) == 16
    _sampled_check(fb, n, n, x, y, edges, edges, tol=1e-6)
    # single tone: exact spike at (f0, f1)
    f0, f1 = 1234, 15000
    i = np.arange(n, dtype=np.int64)
    r0 = np.exp(2j * np.pi * ((f0 * i) % n) / n).astype(np.complex64)
    r1 = np.exp(2j * np.pi * ((f1 * i) % n) / n).astype(np.complex64)
    tone = r0[:, None] * r1[None, :]
    yt = _run(fb, tone)
    assert abs(yt[f0, f1] - n * n) < 1e-4 * n * n
    yt[f0, f1] = 0
    assert np.abs(yt).max() < 1e-4 * n * n


@pytest.mark.parametrize("n0,n1", [(16384, 16384), (8192, 2048), (2048, 2048)])
def test_deterministic_large(fb, n0, n1):
    """Bitwise run-to-run determinism on the persistent TMA path (would expose a race)."""
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    a = fb.fft2d(x)
    b = fb.fft2d(x)
    c = fb.fft2d(x)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(a, c)


def test_delta_closed_form_gpu(fb):
    n0, n1, a, b = 1024, 512, 77, 301
    x = np.zeros((n0, n1), np.complex64)
    x[a, b] = 1
    y = _run(fb, x)
    k0 = np.arange(n0)[:, None]
    k1 = np.arange(n1)[None, :]
    ref = np.exp(-2j * np.pi * ((k0 * a % n0) / n0 + (k1 * b % n1) / n1))
    assert np.abs(y - ref).max() < 2e-6


def test_host_variant(fb):
    x = synth.complex_field(512, 256)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    fb.fb_fft2d_host(xh, yh)
    assert oracle.rel_l2(yh.numpy(), oracle.dft2d(x)) < 5e-7
    fb.fb_fft2d_host(yh, xh, inverse=True)
    assert oracle.rel_l2(xh.numpy(), x) < 5e-7


@pytest.mark.parametrize("batch,n0,n1", [(1, 512, 256), (2, 512, 256), (5, 512, 256), (3, 256, 256),
                                         (2, 360, 100), (2, 1000, 24)])
def test_host_batch_pipeline(fb, batch, n0, n1):
    """Streaming host form: each transform of the batch equals the single-call result bit for
    bit (same kernels, two device slots on two streams) and the oracle within the gate -- also
    for the 256^2 cluster kernel and non-power-of-two sizes (their workspace inside each slot)."""
    xs = np.stack([synth.complex_field(n0, n1, tensor_id=100 + i) for i in range(batch)])
    xb = torch.from_numpy(xs).pin_memory()
    yb = torch.empty_like(xb).pin_memory()
    fb.fb_fft2d_host_batch(xb, yb)
    yh = torch.empty(n0, n1, dtype=torch.complex64).pin_memory()
    for i in range(batch):
        fb.fb_fft2d_host(xb[i].contiguous().pin_memory(), yh)
        assert np.array_equal(yb[i].numpy().view(np.uint32), yh.numpy().view(np.uint32))
        assert oracle.rel_l2(yb[i].numpy(), oracle.dft2d(xs[i])) < 5e-7
    zb = torch.empty_like(xb).pin_memory()
    fb.fb_fft2d_host_batch(yb, zb, inverse=True)
    assert oracle.rel_l2(zb.numpy(), xs) < 5e-7


@pytest.mark.parametrize("n0,n1", [(64, 128), (1, 256), (256, 256)])
def test_nr_fourn_shim(fb, n0, n1):
    """NR fourn conventions: 1-based data/nn, isign=-1 -> exp(-2 pi i), isign=+1 ->
    exp(+2 pi i), both unscaled, in place on the host array."""
    x = synth.complex_field(n0, n1)
    data = np.zeros(2 * n0 * n1 + 1, dtype=np.float32)
    data[1:] = x.view(np.float32).ravel()
    if n0 == 1:
        nn, ndim = np.array([0, n1], dtype=np.uint64), 1
    else:
        nn, ndim = np.array([0, n0, n1], dtype=np.uint64), 2
    fb.fb_nr_fourn(data, nn, ndim, -1)
    y = data[1:].view(np.complex64).reshape(n0, n1)
    assert oracle.rel_l2(y, oracle.dft2d(x)) < 5e-7
    fb.fb_nr_fourn(data, nn, ndim, +1)   # unscaled inverse: returns N * x
    z = data[1:].view(np.complex64).reshape(n0, n1)
    assert oracle.rel_l2(z, (n0 * n1) * x.astype(np.complex128)) < 5e-7
    assert data[0] == 0.0  # the unused NR slot is untouched


@pytest.mark.parametrize("n0,n1", [(512, 64), (512, 256), (1024, 4096), (2048, 2048), (4096, 512)])
def test_pair_plan_matches_plain_plan(fb, n0, n1, monkeypatch):
    """The 2 x n0/2 column split (radix-2 fused into the row pass) against the one-column-pass
    plan (FB_FFT_PAIR=0): both are the same DFT, forward and inverse."""
    monkeypatch.setenv("FB_FFT_PAIR_MAX_LOG2", "12")
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    y_pair = fb.fft2d(x)
    z_pair = fb.ifft2d(y_pair)
    monkeypatch.setenv("FB_FFT_PAIR", "0")
    y_plain = fb.fft2d(x)
    z_plain = fb.ifft2d(y_plain)
    torch.cuda.synchronize()
    assert oracle.rel_l2(y_pair.cpu().numpy(), y_plain.cpu().numpy()) < 5e-7
    assert oracle.rel_l2(z_pair.cpu().numpy(), x.cpu().numpy()) < 5e-7
    assert oracle.rel_l2(z_plain.cpu().numpy(), x.cpu().numpy()) < 5e-7


@pytest.mark.parametrize("n,batch", [(1, 3), (2, 5), (16, 7), (64, 33), (512, 40), (2048, 9), (4096, 4),
                                     (8192, 3), (16384, 2)])
def test_fft1d_batched_vs_oracle(fb, n, batch):
    """fb_fft1d_batched / fb_ifft1d_batched against the 1D DFT definition."""
    xh = synth.complex_field(batch, n)
    x = torch.from_numpy(xh).cuda()
    y = fb.fft1d(x)
    z = fb.fft1d(y, inverse=True)
    w = x.clone()
    fb.fft1d(w, out=w)  # in place
    torch.cuda.synchronize()
    bar = 5e-7 if n <= 4096 else 1e-6
    assert oracle.rel_l2(y.cpu().numpy(), oracle.dft1d_rows(xh)) < bar
    assert oracle.rel_l2(z.cpu().numpy(), xh) < bar
    assert torch.equal(w, y)


def test_fft1d_batched_matches_fft2d_rows(fb):
    """A batch of lines is the row pass of the 2D transform with n0 = 1 per line."""
    xh = synth.complex_field(8, 1024)
    x = torch.from_numpy(xh).cuda()
    y = fb.fft1d(x)
    for b in (0, 7):
        yb = fb.fft2d(x[b:b + 1].contiguous())
        torch.cuda.synchronize()
        assert oracle.rel_l2(y[b:b + 1].cpu().numpy(), yb.cpu().numpy()) < 1e-6


def _real_field(n0, n1):
    return np.ascontiguousarray(synth.complex_field(n0, n1 // 2).view(np.float32).reshape(n0, n1))


@pytest.mark.parametrize("n0,n1", [(1, 2), (2, 2), (4, 8), (64, 128), (256, 256), (512, 64), (2048, 2048),
                                   (8192, 64), (16, 16384)])
def test_rfft2d_vs_oracle(fb, n0, n1):
    """fb_rfft2d / fb_irfft2d (real vibration signals P:149): the Hermitian half of
    the 2D DFT definition of the real input, and the exact inverse."""
    xr = _real_field(n0, n1)
    x = torch.from_numpy(xr).cuda()
    y = fb.rfft2d(x)
    z = fb.irfft2d(y, n1)
    torch.cuda.synchronize()
    h = n1 // 2
    if n0 * n1 <= 2048 * 2048:
        ref = oracle.dft2d(xr.astype(np.complex64))[:, :h + 1]
    else:  # sampled full columns of the oracle
        cols = [0, 1, h // 2, h]
        ref = np.stack([oracle.dft2d_col(xr.astype(np.complex64), c) for c in cols], axis=1)
        y = y[:, cols]
    bar = max(5e-7, 1e-7 * np.log2(n0 * n1))
    assert oracle.rel_l2(y.cpu().numpy(), ref) < bar
    assert oracle.rel_l2(z.cpu().numpy(), xr) < bar


def test_irfft2d_vs_oracle_inverse(fb):
    """The inverse of a Hermitian half equals the oracle's inverse DFT of the Hermitian
    extension (real part; the imaginary part of the oracle result is ~0)."""
    n0, n1 = 64, 32
    X = oracle.dft2d(_real_field(n0, n1).astype(np.complex64))
    half = np.ascontiguousarray(X[:, :n1 // 2 + 1].astype(np.complex64))
    z = fb.irfft2d(torch.from_numpy(half).cuda(), n1)
    torch.cuda.synchronize()
    ref = oracle.dft2d(X.astype(np.complex64), inverse=True)
    assert np.abs(ref.imag).max() < 1e-5
    assert oracle.rel_l2(z.cpu().numpy(), ref.real) < 5e-7


@pytest.mark.parametrize("knobs", [{"FB_FFT_NO_TMA": "1"}, {"FB_FFT_PAIR_TMA": "0"}, {"FB_FFT_ROW_NB": "2"},
                                   {"FB_FFT_COL_NB": "2"}, {"FB_FFT_NO_PDL": "1"}, {"FB_FFT_COL_MAX_LOG2": "10"},
                                   {"FB_FFT_COL_STG": "0"}, {"FB_FFT_COL_STG": "1"}, {"FB_FFT_STAGGER": "0"}])
@pytest.mark.parametrize("n0,n1", [(512, 256), (2048, 128), (4096, 64)])
def test_fft_path_variants_vs_oracle(fb, n0, n1, knobs, monkeypatch):
    """Each kernel path behind an A/B knob (no TMA, plain-kernel pair row pass, forced staging
    buffer counts, no PDL, four-step for shorter columns) computes the same DFT."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    xh = synth.complex_field(n0, n1)
    x = torch.from_numpy(xh).cuda()
    y = fb.fft2d(x)
    z = fb.ifft2d(y)
    torch.cuda.synchronize()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.dft2d(xh)) < 5e-7
    assert oracle.rel_l2(z.cpu().numpy(), xh) < 5e-7


@pytest.mark.parametrize("n0,n1", [(512, 512), (2048, 2048), (8192, 256), (1024, 1024), (2048, 4096), (512, 64),
                                   (4096, 4096), (256, 1024), (64, 2048)])
def test_store_path_and_stagger_bitwise(fb, n0, n1, monkeypatch):
    """The column-output path (exchange buffer + TMA store vs direct register stores), the
    staggered start and the pair step's lane-exchange layout change only how bytes move, not the
    arithmetic: results are bit-identical (forward and inverse)."""
    xh = synth.complex_field(n0, n1)
    x = torch.from_numpy(xh).cuda()
    monkeypatch.setenv("FB_FFT_COL32", "0")  # these knobs select paths of the radix-16 pass
    outs = []
    for knobs in ({}, {"FB_FFT_COL_STG": "0"}, {"FB_FFT_COL_STG": "1"}, {"FB_FFT_STAGGER": "0"},
                  {"FB_FFT_PAIR2": "0"}, {"FB_FFT_PAIR2": "1"}, {"FB_FFT_PAIR2": "2"},
                  {"FB_FFT_COLPAIR": "0"}, {"FB_FFT_COLPAIR": "1"}):
        for k in ("FB_FFT_COL_STG", "FB_FFT_STAGGER", "FB_FFT_PAIR2", "FB_FFT_COLPAIR"):
            monkeypatch.delenv(k, raising=False)
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        y = fb.fft2d(x)
        outs.append(np.concatenate([y.cpu().numpy(), fb.ifft2d(y).cpu().numpy()]))
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))


@pytest.mark.parametrize("n0,n1", [(2048, 2048), (2048, 1024), (2048, 256), (2048, 64)])
def test_radix32_column_pass_vs_oracle(fb, n0, n1, monkeypatch):
    """The 1024-long column pass of the pair plan (2048-row arrays) in its radix-32 one-exchange
    form (fft_col1024_kernel) and in the radix-16 form (FB_FFT_COL32=0): both match the oracle
    within the 5e-7 gate, forward and inverse (conj + exact 1/(n0 n1) scale in its epilogue),
    and the radix-32 form is bitwise deterministic and in-place safe."""
    xh = synth.complex_field(n0, n1)
    ref = oracle.dft2d(xh)
    x = torch.from_numpy(xh).cuda()
    outs = {}
    for v in ("1", "0"):
        monkeypatch.setenv("FB_FFT_COL32", v)
        y = fb.fft2d(x)
        z = fb.ifft2d(y)
        y2 = fb.fft2d(x)
        xi = x.clone()
        fb.fft2d(xi, out=xi)
        torch.cuda.synchronize()
        assert torch.equal(y, y2) and torch.equal(y, xi)
        assert oracle.rel_l2(y.cpu().numpy(), ref) < 5e-7, v
        assert oracle.rel_l2(z.cpu().numpy(), xh) < 5e-7, v
        outs[v] = y.cpu().numpy()
    assert oracle.rel_l2(outs["1"], outs["0"]) < 5e-7


@pytest.mark.parametrize("mixed", ["1", "0", "2"])
@pytest.mark.parametrize("n0,n1", [(3, 5), (7, 64), (1, 999), (1000, 1), (100, 36), (360, 480), (12, 8191),
                                   (2048, 1000), (625, 243), (2401, 6), (10, 6561), (3125, 5), (14, 8000),
                                   (4200, 6), (6, 4200), (1000, 24), (3, 7776)])
def test_non_power_of_two_vs_oracle(fb, n0, n1, mixed, monkeypatch):
    """sizes that are not powers of two against the full oracle, forward and
    inverse, within the north_star bar 1e-5 log2(n0 n1); in place equals out of place.  Lines
    whose length factors into 2, 3, 5, 7 run the mixed-radix Stockham kernel (FB_FFT_MIXED=1,
    radix 8/4/2/3/5/7 stages; =2 also runs the columns in place, C at a time), the others
    (999 = 27 * 37, the prime 8191) and every line with FB_FFT_MIXED=0 Bluestein's chirp-z over
    the power-of-two passes (fb_bluestein.cu)."""
    monkeypatch.setenv("FB_FFT_MIXED", mixed)
    x = synth.complex_field(n0, n1, tensor_id=7)
    ref = oracle.dft2d(x)
    y = _run(fb, x)
    e = oracle.rel_l2(y, ref)
    z = _run(fb, y, inverse=True)
    ei = oracle.rel_l2(z, oracle.dft2d(y, inverse=True))
    print(f"{n0}x{n1}: forward {e:.2e} inverse {ei:.2e}")
    assert e < _bar(n0, n1) and ei < _bar(n0, n1), (e, ei)
    assert e < 2e-6  # the measured level (FP32 chirp-z): well inside the bar
    assert np.array_equal(_run(fb, x, inplace=True), y)


@pytest.mark.parametrize("mixed", ["1", "0", "2"])
def test_non_power_of_two_square_tone(fb, mixed, monkeypatch):
    """4200 x 4200 (2^3 3 5^2 7): square with columns longer than 4096, one column per CTA in the
    mixed-radix kernel; a single tone must land in one bin with the rest at rounding level."""
    monkeypatch.setenv("FB_FFT_MIXED", mixed)
    n = 4200
    f0, f1 = 1234, 4001
    i0 = torch.arange(n, dtype=torch.float64, device="cuda")[:, None]
    i1 = torch.arange(n, dtype=torch.float64, device="cuda")[None, :]
    ph = 2 * np.pi * (torch.remainder(f0 * i0, n) / n + torch.remainder(f1 * i1, n) / n)
    tone = torch.polar(torch.ones_like(ph), ph).to(torch.complex64)
    y = fb.fft2d(tone)
    peak = complex(y[f0, f1].item())
    y[f0, f1] = 0
    rest = float(y.abs().max().item())
    assert abs(peak - n * n) < 1e-4 * n * n and rest < 1e-4 * n * n, (peak, rest)


def test_non_power_of_two_closed_forms(fb):
    """Tone and delta closed forms at a non-power-of-two size (3 * 5 * 7 * 11 x 2 * 3^4)."""
    n0, n1 = 1155, 162
    f0, f1 = 77, 13
    i0 = np.arange(n0)[:, None]
    i1 = np.arange(n1)[None, :]
    tone = np.exp(2j * np.pi * (((f0 * i0) % n0) / n0 + ((f1 * i1) % n1) / n1)).astype(np.complex64)
    yt = _run(fb, tone)
    assert abs(yt[f0, f1] - n0 * n1) < 1e-4 * n0 * n1
    yt[f0, f1] = 0
    assert np.abs(yt).max() < 1e-4 * n0 * n1
    d = np.zeros((n0, n1), np.complex64)
    a, b = 401, 99
    d[a, b] = 1
    yd = _run(fb, d)
    ref = np.exp(-2j * np.pi * (((i0 * a) % n0) / n0 + ((i1 * b) % n1) / n1))
    assert np.abs(yd - ref).max() < 1e-5


@pytest.mark.parametrize("inverse", [False, True])
def test_row16384_cluster_kernel_bitwise(fb, inverse, monkeypatch):
    """FB_FFT_ROW16K=2: each 16384-long line split over a CTA pair (stage-A outputs exchanged
    through distributed shared memory, two or three half-line CTAs per SM) runs the per-element
    operations of the one-CTA-per-line kernel, so 1D rows (conj/scale of the inverse included)
    and a 2D transform with 16384-long rows are bitwise equal to it."""
    n0, n1 = 300, 16384
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    y1 = fb.fft1d(x, inverse=inverse)
    x2 = torch.from_numpy(synth.complex_field(64, 16384)).cuda()
    z1 = fb.fft2d(x2, inverse=inverse)
    monkeypatch.setenv("FB_FFT_ROW16K", "2")
    y2 = fb.fft1d(x, inverse=inverse)
    z2 = fb.fft2d(x2, inverse=inverse)
    monkeypatch.setenv("FB_FFT_ROW16K_CPS", "3")
    y3 = fb.fft1d(x, inverse=inverse)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2) and torch.equal(z1, z2) and torch.equal(y1, y3)


def test_longrow_kernel_matches_plain_kernel(fb, monkeypatch):
    """16384-long rows: the radix-16 persistent half-prefetching kernel (FB_FFT_ROW16K=0) and the
    plain kernel run the same per-line arithmetic (bit for bit); the default 32 x 32 x 16
    four-step kernel (fft_row16384_kernel) is a different factorisation: it matches the oracle
    on sampled rows like both, and is bitwise deterministic."""
    n0, n1 = 48, 16384
    xh = synth.complex_field(n0, n1)
    x = torch.from_numpy(xh).cuda()
    y4 = fb.fft1d(x)
    y4b = fb.fft1d(x)
    monkeypatch.setenv("FB_FFT_ROW16K", "0")
    y1 = fb.fft1d(x)
    monkeypatch.setenv("FB_FFT_LONGROW", "0")
    y0 = fb.fft1d(x)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(y4, y4b)
    for r in (0, 1, 47):
        ref = oracle.dft1d_rows(xh[r:r + 1])
        assert oracle.rel_l2(y1[r:r + 1].cpu().numpy(), ref) < 1e-6
        assert oracle.rel_l2(y4[r:r + 1].cpu().numpy(), ref) < 1e-6
