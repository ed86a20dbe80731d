"""GPU parity of the LU block (fb_lu through the C ABI) against the LU oracle.

Pivots (an argmax decided in FP64 on both sides) must match exactly; the factors must match
the oracle within 1e-11 relative (different but equally valid FP64 summation order in the
blocked trailing updates: the bound is a few n*eps times the growth of the factors), and the
reconstruction P A = L U must hold to 1e-13 relative."""
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


def _check(fb, A, tol=1e-11):
    LU, ipiv, info = fb.lu(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    LU, ipiv, info = LU.cpu().numpy(), ipiv.cpu().numpy(), int(info.item())
    LU_o, ipiv_o, info_o = oracle.lu(A)
    assert info == info_o
    assert np.array_equal(ipiv, ipiv_o)
    assert oracle.rel_l2(LU, LU_o) < tol
    n = A.shape[0]
    L = np.tril(LU, -1) + np.eye(n)
    U = np.triu(LU)
    p = oracle.lu_permutation(ipiv)
    assert np.linalg.norm(A[p] - L @ U) / np.linalg.norm(A) < 1e-13
    return LU, ipiv


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 9, 33, 100, 256, 511])
def test_lu_random_vs_oracle(fb, n):
    A = synth.real_matrix(n, n, synth.TID_GEMM_A, dtype=np.float64) if n > 1 else np.array([[0.5]])
    _check(fb, np.ascontiguousarray(A))


def test_lu_hand_example(fb):
    A = np.array([[1.0, 2, 3], [4, 5, 6], [7, 8, 10]])
    LU, ipiv = _check(fb, A, tol=1e-15)
    assert list(ipiv) == [2, 2, 2]


def test_lu_orthogonal_2048(fb):
    """The paper's workload: LU of a 2048x2048 orthogonal matrix; |det Q| = 1."""
    Q = synth.dct2_matrix(2048)
    LU, ipiv = _check(fb, Q)
    assert abs(abs(np.prod(np.diag(LU))) - 1.0) < 1e-10


def test_lu_2048_random(fb):
    A = synth.real_matrix(2048, 2048, synth.TID_GEMM_A, dtype=np.float64)
    _check(fb, A)


def test_lu_4096_large_panel_path(fb):
    n = 3000
    A = synth.real_matrix(n, n, synth.TID_GEMM_B, dtype=np.float64)
    _check(fb, A)


def test_lu_singular(fb):
    A = np.array([[0.0, 1.0, 2.0], [0.0, 2.0, 1.0], [0.0, 3.0, 5.0]])
    LU, ipiv, info = fb.lu(torch.from_numpy(A).cuda())
    torch.cuda.synchronize()
    assert int(info.item()) == 1
    LU_o, ipiv_o, info_o = oracle.lu(A)
    assert info_o == 1 and np.array_equal(ipiv.cpu().numpy(), ipiv_o)
    assert np.allclose(LU.cpu().numpy(), LU_o, atol=1e-15)


def test_lu_deterministic(fb):
    A = torch.from_numpy(synth.real_matrix(1024, 1024, synth.TID_GEMM_A, dtype=np.float64)).cuda()
    a = fb.lu(A)[0]
    b = fb.lu(A)[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)


def test_lu_repeated_outside_pivot_row(fb):
    """A row outside a panel chosen as pivot at two consecutive steps (exercises the swap
    replay of the row-swap kernel): the large entries live in the same far row."""
    n = 40
    A = synth.real_matrix(n, n, synth.TID_GEMM_B, dtype=np.float64) * 0.01
    A[30, 0] = 50.0   # step 0 pivots row 30 -> old row 0 moves to row 30
    A[0, 1] = 40.0    # ... which (after the rank-1 update) holds the step-1 pivot again
    A[30, 1] = 1.0
    _check(fb, np.ascontiguousarray(A))


@pytest.mark.parametrize("knobs", [{"FB_LU_GRAPH": "0"}, {"FB_LU_TMA": "0"}, {"FB_LU_RANK_SIMT": "0"},
                                   {"FB_LU_SERIAL": "1", "FB_LU_GRAPH": "0"}, {"FB_LU_LOOKAHEAD": "0"}])
@pytest.mark.parametrize("n", [40, 777, 2048])
def test_lu_schedule_variants(fb, n, knobs, monkeypatch):
    """Every schedule / kernel variant behind an A/B knob (stream-ordered instead of graph,
    cp.async instead of TMA panel, DMMA instead of streaming rank update, wide parts on one
    stream, no look-ahead) gives the same pivots and factors within the oracle bar."""
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    _check(fb, synth.real_matrix(n, n, synth.TID_GEMM_A).astype(np.float64))


def test_lu_graph_replay_reuses_buffers(fb):
    """The cached graph replays on the same buffers with new contents (the key is the
    pointers and sizes, not the data)."""
    n = 1000
    buf = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    ipiv = torch.empty(n, dtype=torch.int32, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    for seed_tid in (synth.TID_GEMM_A, synth.TID_GEMM_B, synth.TID_NOISE):
        A = synth.real_matrix(n, n, seed_tid).astype(np.float64)
        buf.copy_(torch.from_numpy(A))
        fb.fb_lu(buf, ipiv, info)
        torch.cuda.synchronize()
        LU_o, ipiv_o, _ = oracle.lu(A)
        assert np.array_equal(ipiv.cpu().numpy(), ipiv_o)
        assert oracle.rel_l2(buf.cpu().numpy(), LU_o) < 1e-11
