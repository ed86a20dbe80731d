"""The multi-GPU entry points (NCCL communicator, slab FFT, row-block GEMM) on the one GPU this
build has: world size 1 exercises fb_comm_init, the NCCL device communicator, the symmetric
window and LSA barriers of the fused transpose, the NCCL path (ncclAlltoAll / ncclBroadcast)
and the column passes.  The P > 1 peer addressing of the fused transpose is covered by
fb_fft2d_slab_model, which runs the P ranks' kernels one after another on this GPU with P
local windows (no rank waits on another)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import __graft_entry__
    __graft_entry__.build_lib()
    import paper_2004_09883_b200 as fb
    torch.cuda.set_device(0)
    fb.fb_init(0)
    comm = fb.Comm(0, 1, 0)
    yield fb, comm
    comm.destroy()


@pytest.mark.parametrize("n0,n1", [(256, 256), (2048, 2048), (16384, 64), (64, 4096)])
def test_slab_world1_equals_fft2d(env, n0, n1):
    fb, comm = env
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    y = torch.empty_like(x)
    comm.fb_fft2d_slab(x, y, n0, n1)
    ref = fb.fft2d(x)
    torch.cuda.synchronize()
    # same definition; the single-GPU call may use a different column split (pair plan)
    assert oracle.rel_l2(y.cpu().numpy(), ref.cpu().numpy()) < 5e-7
    z = torch.empty_like(x)
    comm.fb_ifft2d_slab(y, z, n0, n1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(z.cpu().numpy(), x.cpu().numpy()) < 5e-7


def test_slab_world1_vs_oracle(env):
    fb, comm = env
    n0, n1 = 512, 256
    xh = synth.complex_field(n0, n1)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty_like(x)
    comm.fb_fft2d_slab(x, y, n0, n1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(y.cpu().numpy(), oracle.dft2d(xh)) < 5e-7


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
def test_rowblock_world1(env, dt):
    fb, comm = env
    m, n, k = 512, 384, 256
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(dt).cuda()
    B = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(dt).cuda()
    C = torch.empty(m, n, dtype=dt, device="cuda")
    comm.fb_matmul_rowblock(A, B, C, root=0)
    ref = fb.matmul(A, B)
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    bar = 1e-5 if dt == torch.float32 else 1e-12
    assert oracle.rel_l2(C.cpu().numpy(), oracle.matmul(A.cpu().numpy(), B.cpu().numpy())) < bar


def test_comm_validation(env):
    fb, comm = env
    x = torch.zeros(6, 8, dtype=torch.complex64, device="cuda")
    with pytest.raises(fb.FbError):
        comm.fb_fft2d_slab(x, x, 6, 8)  # not a power of two


def test_world1_is_fused(env):
    fb, comm = env
    assert comm.fused, comm.fused_detail


def test_fused_equals_nccl_path_bitwise(env, monkeypatch):
    fb, comm = env
    monkeypatch.setenv("FB_SLAB_FUSED", "0")
    plain = fb.Comm(0, 1, 0)
    try:
        assert not plain.fused and "FB_SLAB_FUSED" in plain.fused_detail
        for n0, n1 in [(256, 256), (2048, 1024), (8192, 64)]:
            x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
            y1, y2 = torch.empty_like(x), torch.empty_like(x)
            comm.fb_fft2d_slab(x, y1, n0, n1)
            plain.fb_fft2d_slab(x, y2, n0, n1)
            z1, z2 = torch.empty_like(x), torch.empty_like(x)
            comm.fb_ifft2d_slab(y1, z1, n0, n1)
            plain.fb_ifft2d_slab(y2, z2, n0, n1)
            torch.cuda.synchronize()
            assert torch.equal(y1, y2) and torch.equal(z1, z2), (n0, n1)
    finally:
        plain.destroy()


def _assemble(y, P, n0, n1):
    """[P][n0][n1/P] column slabs -> n0 x n1."""
    return y.view(P, n0, n1 // P).permute(1, 0, 2).reshape(n0, n1)


@pytest.mark.parametrize("n0,n1", [(256, 256), (2048, 2048), (64, 4096), (8192, 64), (16, 8)])
def test_fused_model_all_P_bitwise(env, n0, n1):
    """The fused transpose's peer addressing for P = 2, 4, 8 virtual ranks: every P computes the
    same per-line arithmetic, so the assembled result equals P = 1 bit for bit, and P = 1
    equals the real world-size-1 fused call."""
    fb, comm = env
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    ref = torch.empty_like(x)
    comm.fb_fft2d_slab(x, ref, n0, n1)
    for P in (1, 2, 4, 8):
        if n0 % P or n1 % P:
            continue
        y = torch.empty(n0 * n1, dtype=torch.complex64, device="cuda")
        fb.fb_fft2d_slab_model(P, x, y, n0, n1)
        z = torch.empty_like(x)
        fb.fb_fft2d_slab_model(P, z, y, n0, n1, inverse=True)
        torch.cuda.synchronize()
        assert torch.equal(_assemble(y, P, n0, n1), ref), P
        assert oracle.rel_l2(z.cpu().numpy(), x.cpu().numpy()) < 5e-7, P
        if P == 1:
            zr = torch.empty_like(x)
            comm.fb_ifft2d_slab(ref, zr, n0, n1)
            torch.cuda.synchronize()
            assert torch.equal(z, zr)
        else:
            z1 = torch.empty_like(x)
            fb.fb_fft2d_slab_model(1, z1, y.view(P, n0, n1 // P).permute(1, 0, 2).reshape(-1).contiguous(), n0, n1,
                                   inverse=True)
            torch.cuda.synchronize()
            assert torch.equal(z, z1), P


@pytest.mark.parametrize("row16k", ["1", "2"])
def test_fused_model_16384_rows_bitwise(env, row16k, monkeypatch):
    """16384-long rows through the per-peer output map (the slab transpose's row pass in the
    one-CTA-per-line and the CTA-pair kernels): P = 2, 4, 8 assemble to P = 1 bit for bit."""
    fb, _ = env
    monkeypatch.setenv("FB_FFT_ROW16K", row16k)
    n0, n1 = 64, 16384
    x = torch.from_numpy(synth.complex_field(n0, n1)).cuda()
    ys = {}
    for P in (1, 2, 4, 8):
        y = torch.empty(n0 * n1, dtype=torch.complex64, device="cuda")
        fb.fb_fft2d_slab_model(P, x, y, n0, n1)
        ys[P] = _assemble(y, P, n0, n1)
    torch.cuda.synchronize()
    for P in (2, 4, 8):
        assert torch.equal(ys[P], ys[1]), P


def test_fused_model_vs_oracle(env):
    fb, _ = env
    n0, n1, P = 512, 256, 4
    xh = synth.complex_field(n0, n1)
    x = torch.from_numpy(xh).cuda()
    y = torch.empty(n0 * n1, dtype=torch.complex64, device="cuda")
    fb.fb_fft2d_slab_model(P, x, y, n0, n1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(_assemble(y, P, n0, n1).cpu().numpy(), oracle.dft2d(xh)) < 5e-7


@pytest.mark.parametrize("dt", [torch.float32, torch.float64])
@pytest.mark.parametrize("panel", ["64", "100", "0", "512"])
def test_rowblock_panel_broadcast_world1(env, panel, dt, monkeypatch):
    """The row-block GEMM broadcasts B in N-column panels on the communicator's stream and runs
    the GEMM of panel j (full K) as soon as it lands, while panel j+1 is on the wire (SURVEY
    8(a) G5); the root packs each panel into a reused workspace slot.  The product is bitwise the
    plain fb_matmul product (same per-element arithmetic), ragged last panel included, and the
    root's B is left unchanged."""
    fb, comm = env
    monkeypatch.setenv("FB_ROWBLOCK_PANEL", panel)
    m, n, k = 256, 1192, 300
    A = torch.from_numpy(synth.real_matrix(m, k, synth.TID_GEMM_A)).to(dt).cuda()
    B = torch.from_numpy(synth.real_matrix(k, n, synth.TID_GEMM_B)).to(dt).cuda()
    B0 = B.clone()
    C = torch.empty(m, n, dtype=dt, device="cuda")
    for _ in range(2):  # the second call reuses the slots and events
        comm.fb_matmul_rowblock(A, B, C, root=0)
    ref = fb.matmul(A, B0)
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    assert torch.equal(B, B0)


def test_fused_model_config3_full_size(env):
    """configs[3] at its full size: the fused slab transpose's addressing for P = 2 and 8 virtual
    ranks on the 16384^2 problem, bitwise against P = 1 (the same per-line kernels), and P = 1
    against the single-GPU 2D FFT (different column plan: tolerance)."""
    fb, comm = env
    n = 16384
    x = torch.from_numpy(synth.complex_field(n, n)).cuda()
    y1 = torch.empty(n * n, dtype=torch.complex64, device="cuda")
    fb.fb_fft2d_slab_model(1, x, y1, n, n)
    y1 = y1.view(n, n)
    for P in (2, 8):
        y = torch.empty(n * n, dtype=torch.complex64, device="cuda")
        fb.fb_fft2d_slab_model(P, x, y, n, n)
        torch.cuda.synchronize()
        assert torch.equal(_assemble(y, P, n, n), y1), P
        del y
    ref = fb.fft2d(x)
    torch.cuda.synchronize()
    d = (y1 - ref).abs().pow(2).sum().sqrt() / ref.abs().pow(2).sum().sqrt()
    assert float(d) < 1e-6
