"""Host-side simulation of the slab-sharded 2D FFT data contract (reading R8).

P ranks are simulated in numpy with the SAME index maps the CUDA passes use
(csrc/fb_comm.cu): the row pass stores element k of local row i at
send[k // (n1/P)][i][k % (n1/P)]; ncclAlltoAll delivers block d of rank s to recv[s] of
rank d; the received buffer is the natural n0 x (n1/P) column strip.  numpy.fft supplies the
1D transforms (this test checks the data movement, not the arithmetic).
"""
import numpy as np
import pytest

import paper_2004_09883_b200 as fb


def _alltoall(sends):
    P = len(sends)
    return [np.stack([sends[s][d] for s in range(P)]) for d in range(P)]


def slab_forward(x, P):
    n0, n1 = x.shape
    rows, cols = n0 // P, n1 // P
    sends = []
    for r in range(P):
        r0, r1 = fb.slab_rows(r, P, n0)
        y = np.fft.fft(x[r0:r1], axis=1)                    # row pass
        send = np.empty((P, rows, cols), dtype=y.dtype)
        for k in range(n1):                                  # the pass's store map
            send[k // cols, :, k % cols] = y[:, k]
        sends.append(send)
    recvs = _alltoall(sends)
    out = []
    for r in range(P):
        strip = recvs[r].reshape(n0, cols)                   # natural column strip
        out.append(np.fft.fft(strip, axis=0))                # column pass
    return out


def slab_inverse(ycols, n0, n1, P):
    rows, cols = n0 // P, n1 // P
    sends = []
    for r in range(P):
        z = np.fft.ifft(ycols[r], axis=0)                    # column pass (n0 x cols)
        sends.append(z.reshape(P, rows, cols))               # rows of peer d are contiguous
    recvs = _alltoall(sends)
    out = []
    for r in range(P):
        line = np.empty((rows, n1), dtype=recvs[r].dtype)
        for k in range(n1):                                  # the pass's load map
            line[:, k] = recvs[r][k // cols, :, k % cols]
        out.append(np.fft.ifft(line, axis=1))                # row pass
    return out


@pytest.mark.parametrize("n0,n1,P", [(16, 16, 2), (16, 16, 4), (32, 16, 8), (64, 128, 8), (8, 8, 8),
                                     (128, 32, 2), (16, 64, 1)])
def test_slab_contract(n0, n1, P):
    rng = np.random.default_rng(n0 * n1 * P)
    x = rng.standard_normal((n0, n1)) + 1j * rng.standard_normal((n0, n1))
    Y = np.fft.fft2(x)
    ycols = slab_forward(x, P)
    for r in range(P):
        c0, c1 = fb.slab_cols(r, P, n1)
        assert np.allclose(ycols[r], Y[:, c0:c1], atol=1e-9)
    back = slab_inverse(ycols, n0, n1, P)
    for r in range(P):
        r0, r1 = fb.slab_rows(r, P, n0)
        assert np.allclose(back[r], x[r0:r1], atol=1e-12)


def test_partition_errors():
    with pytest.raises(ValueError):
        fb.slab_rows(0, 3, 16)
    assert fb.slab_cols(3, 4, 64) == (48, 64)
