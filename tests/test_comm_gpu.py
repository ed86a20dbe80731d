"""The multi-GPU entry points (NCCL communicator, slab FFT, row-block GEMM) on the one GPU this
build has: world size 1 exercises fb_comm_init, the fused pack/unpack maps, ncclAlltoAll /
ncclBroadcast and the column passes; results must equal the single-GPU calls bit for bit
(same kernels, same order) and match the oracle."""
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
