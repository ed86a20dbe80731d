"""Python binding for libfb.so -- the B200-native function blocks of arXiv 2004.09883.

Argument marshalling only: every step of the hot path runs in libfb's CUDA kernels
(csrc/).  torch is used for device memory, streams and torch.distributed (plumbing).
There is NO CPU fallback: if libfb.so is missing or the device is not sm_100, calls raise.

The functions carry the C-ABI names of include/fb.h (fb_fft2d, fb_ifft2d, fb_matmul,
fb_fft2d_host, fb_matmul_host, fb_fft2d_slab, fb_ifft2d_slab, fb_matmul_rowblock, ...);
``fft2d``/``ifft2d``/``matmul`` are conveniences that allocate outputs/workspaces.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FB_LIB", os.path.join(_HERE, "libfb.so"))  # FB_LIB: experiment builds

FB_F32 = 0
FB_F64 = 1
_STATUS = {0: "FB_OK", 1: "FB_ERR_INVALID_VALUE", 2: "FB_ERR_UNSUPPORTED_SIZE", 3: "FB_ERR_MISALIGNED",
           4: "FB_ERR_WORKSPACE", 5: "FB_ERR_NOT_INITIALIZED", 6: "FB_ERR_CUDA", 7: "FB_ERR_NCCL",
           8: "FB_ERR_ARCH"}

# every symbol include/fb.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fb_version", "fb_status_string", "fb_last_error_detail", "fb_launch_count", "fb_reload_knobs", "fb_init",
    "fb_fft2d_workspace_bytes", "fb_fft2d", "fb_ifft2d", "fb_fft1d_batched", "fb_ifft1d_batched",
    "fb_gemm_workspace_bytes", "fb_gemm", "fb_rfft2d_workspace_bytes", "fb_rfft2d", "fb_irfft2d",
    "fb_matmul_bf16_workspace_bytes", "fb_matmul_bf16",
    "fb_matmul_workspace_bytes", "fb_matmul", "fb_tf32_split", "fb_matmul_3xtf32_presplit",
    "fb_fft2d_host_workspace_bytes", "fb_fft2d_host", "fb_fft2d_host_batch_workspace_bytes",
    "fb_fft2d_host_batch", "fb_matmul_host_workspace_bytes", "fb_matmul_host",
    "fb_comm_unique_id_bytes", "fb_comm_unique_id", "fb_comm_init", "fb_comm_destroy", "fb_comm_rank",
    "fb_comm_size", "fb_fft2d_slab_workspace_bytes", "fb_fft2d_slab", "fb_ifft2d_slab",
    "fb_comm_fused", "fb_comm_fused_detail", "fb_fft2d_slab_model",
    "fb_matmul_rowblock_workspace_bytes", "fb_matmul_rowblock", "fb_nr_fourn",
    "fb_lu_workspace_bytes", "fb_lu",
]


class FbError(RuntimeError):
    def __init__(self, fn, status, detail):
        super().__init__(f"{fn}: {_STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfb.so (build it first with __graft_entry__.build() / _build.py)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, ci, sz, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_uint64
    sig = {
        "fb_version": ([], ci),
        "fb_status_string": ([ci], ctypes.c_char_p),
        "fb_last_error_detail": ([], ctypes.c_char_p),
        "fb_launch_count": ([], u64),
        "fb_reload_knobs": ([], None),
        "fb_init": ([ci], ci),
        "fb_fft2d_workspace_bytes": ([i64, i64], sz),
        "fb_fft2d": ([vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_ifft2d": ([vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_fft1d_batched": ([vp, vp, i64, i64, vp], ci),
        "fb_rfft2d_workspace_bytes": ([i64, i64], sz),
        "fb_rfft2d": ([vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_irfft2d": ([vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_ifft1d_batched": ([vp, vp, i64, i64, vp], ci),
        "fb_matmul_workspace_bytes": ([ci, i64, i64, i64], sz),
        "fb_gemm_workspace_bytes": ([ci, ci, ci, i64, i64, i64], sz),
        "fb_matmul_bf16_workspace_bytes": ([ci, i64, i64, i64], sz),
        "fb_matmul_bf16": ([i64, i64, i64, vp, i64, vp, i64, ci, vp, i64, vp, sz, vp], ci),
        "fb_gemm": ([ci, ci, ci, i64, i64, i64, ctypes.c_double, vp, i64, vp, i64, ctypes.c_double, vp, i64, vp,
                     sz, vp], ci),
        "fb_matmul": ([ci, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp], ci),
        "fb_tf32_split": ([ci, i64, i64, vp, i64, vp, vp, i64, vp], ci),
        "fb_matmul_3xtf32_presplit": ([i64, i64, i64, vp, vp, i64, vp, vp, i64, vp, i64, vp], ci),
        "fb_fft2d_host_workspace_bytes": ([i64, i64], sz),
        "fb_fft2d_host": ([vp, vp, i64, i64, ci, vp, sz, vp], ci),
        "fb_fft2d_host_batch_workspace_bytes": ([i64, i64], sz),
        "fb_fft2d_host_batch": ([vp, vp, i64, i64, i64, ci, vp, sz, vp], ci),
        "fb_matmul_host_workspace_bytes": ([ci, i64, i64, i64], sz),
        "fb_matmul_host": ([ci, i64, i64, i64, vp, vp, vp, vp, sz, vp], ci),
        "fb_comm_unique_id_bytes": ([], sz),
        "fb_comm_unique_id": ([vp], ci),
        "fb_comm_init": ([ctypes.POINTER(vp), ci, ci, vp, ci], ci),
        "fb_comm_destroy": ([vp], ci),
        "fb_comm_rank": ([vp], ci),
        "fb_comm_size": ([vp], ci),
        "fb_fft2d_slab_workspace_bytes": ([ci, i64, i64], sz),
        "fb_fft2d_slab": ([vp, vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_ifft2d_slab": ([vp, vp, vp, i64, i64, vp, sz, vp], ci),
        "fb_comm_fused": ([vp], ci),
        "fb_comm_fused_detail": ([vp], ctypes.c_char_p),
        "fb_fft2d_slab_model": ([ci, ci, vp, vp, i64, i64, vp, vp, sz, vp], ci),
        "fb_matmul_rowblock_workspace_bytes": ([ci, ci, i64, i64, i64], sz),
        "fb_matmul_rowblock": ([vp, ci, i64, i64, i64, vp, i64, vp, i64, ci, vp, i64, vp, sz, vp], ci),
        "fb_nr_fourn": ([vp, vp, ci, ci], ci),
        "fb_lu_workspace_bytes": ([ci, i64], sz),
        "fb_lu": ([ci, i64, vp, i64, vp, vp, vp, sz, vp], ci),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(fn: str, status: int):
    if status != 0:
        detail = lib().fb_last_error_detail().decode(errors="replace")
        raise FbError(fn, status, detail)


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def launch_count() -> int:
    return int(lib().fb_launch_count())


def fb_reload_knobs():
    """Re-read the FB_* A/B knobs from the environment (libfb reads them once per process)."""
    lib().fb_reload_knobs()


def fb_init(device: int = 0):
    _check("fb_init", lib().fb_init(device))


# ------------------------------------------------------------------ workspace cache (plumbing)


def _workspace(nbytes: int, device, stream=None) -> torch.Tensor | None:
    return None if nbytes == 0 else _workspace_named(nbytes, device, "ws", stream)


# ------------------------------------------------------------------ Fourier block
def _fft_check(x: torch.Tensor):
    if x.dtype != torch.complex64 or not x.is_cuda or x.dim() != 2 or not x.is_contiguous():
        raise ValueError("expected a contiguous 2D complex64 CUDA tensor")


def fb_fft2d(x: torch.Tensor, y: torch.Tensor, ws: torch.Tensor | None = None, stream=None):
    n0, n1 = x.shape
    _check("fb_fft2d", lib().fb_fft2d(_ptr(x), _ptr(y), n0, n1, _ptr(ws), 0 if ws is None else ws.numel(),
                                      _stream(stream)))


def fb_ifft2d(x: torch.Tensor, y: torch.Tensor, ws: torch.Tensor | None = None, stream=None):
    n0, n1 = x.shape
    _check("fb_ifft2d", lib().fb_ifft2d(_ptr(x), _ptr(y), n0, n1, _ptr(ws), 0 if ws is None else ws.numel(),
                                        _stream(stream)))


def fft2d(x: torch.Tensor, out: torch.Tensor | None = None, inverse: bool = False, stream=None) -> torch.Tensor:
    """2D DFT (sign -1, unscaled) or inverse (sign +1, 1/(n0 n1)) of a complex64 CUDA tensor."""
    _fft_check(x)
    out = torch.empty_like(x) if out is None else out
    _fft_check(out)
    n0, n1 = x.shape
    ws = _workspace(lib().fb_fft2d_workspace_bytes(n0, n1), x.device, stream)
    (fb_ifft2d if inverse else fb_fft2d)(x, out, ws, stream)
    return out


def fft1d(x: torch.Tensor, out: torch.Tensor | None = None, inverse: bool = False, stream=None) -> torch.Tensor:
    """1D DFT of every row of a [batch, n] complex64 CUDA tensor (fb_fft1d_batched)."""
    _fft_check(x)
    out = torch.empty_like(x) if out is None else out
    _fft_check(out)
    b, n = x.shape
    f = lib().fb_ifft1d_batched if inverse else lib().fb_fft1d_batched
    _check("fb_fft1d_batched", f(_ptr(x), _ptr(out), n, b, _stream(stream)))
    return out


def rfft2d(x: torch.Tensor, stream=None) -> torch.Tensor:
    """Hermitian half [n0, n1/2+1] (complex64) of the 2D DFT of a real float32 CUDA tensor."""
    if x.dtype != torch.float32 or not x.is_cuda or x.dim() != 2 or not x.is_contiguous():
        raise ValueError("expected a contiguous 2D float32 CUDA tensor")
    n0, n1 = x.shape
    y = torch.empty(n0, n1 // 2 + 1, dtype=torch.complex64, device=x.device)
    ws = _workspace_named(lib().fb_rfft2d_workspace_bytes(n0, n1), x.device, "rfft", stream)
    _check("fb_rfft2d", lib().fb_rfft2d(_ptr(x), _ptr(y), n0, n1, _ptr(ws), ws.numel(), _stream(stream)))
    return y


def irfft2d(y: torch.Tensor, n1: int, stream=None) -> torch.Tensor:
    """Real [n0, n1] inverse of rfft2d (scaled 1/(n0 n1))."""
    if y.dtype != torch.complex64 or not y.is_cuda or y.dim() != 2 or not y.is_contiguous():
        raise ValueError("expected a contiguous 2D complex64 CUDA tensor")
    n0 = y.shape[0]
    x = torch.empty(n0, n1, dtype=torch.float32, device=y.device)
    ws = _workspace_named(lib().fb_rfft2d_workspace_bytes(n0, n1), y.device, "rfft", stream)
    _check("fb_irfft2d", lib().fb_irfft2d(_ptr(y), _ptr(x), n0, n1, _ptr(ws), ws.numel(), _stream(stream)))
    return x


def ifft2d(x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    return fft2d(x, out, inverse=True, stream=stream)


# ------------------------------------------------------------------ matrix block
def matmul_bf16(A: torch.Tensor, B: torch.Tensor, b_transposed: bool = False, out: torch.Tensor | None = None,
                stream=None) -> torch.Tensor:
    """float32 C = A @ B for bfloat16 A [m, k] and B [k, n] (or B^T [n, k] when b_transposed)."""
    if A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise ValueError("matmul_bf16 expects bfloat16 operands")
    m, k = A.shape
    n = B.shape[0] if b_transposed else B.shape[1]
    C = torch.empty(m, n, dtype=torch.float32, device=A.device) if out is None else out
    ws = _workspace_named(lib().fb_matmul_bf16_workspace_bytes(int(b_transposed), m, n, k), A.device, "bf16", stream)
    _check("fb_matmul_bf16", lib().fb_matmul_bf16(m, n, k, _ptr(A), A.stride(0), _ptr(B), B.stride(0),
                                                  int(b_transposed), _ptr(C), C.stride(0), _ptr(ws), ws.numel(),
                                                  _stream(stream)))
    return C


def gemm(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor | None = None, alpha: float = 1.0, beta: float = 0.0,
         trans_a: bool = False, trans_b: bool = False, stream=None) -> torch.Tensor:
    """C = alpha op(A) op(B) + beta C (fb_gemm); float32 (3xTF32) or float64 (DMMA)."""
    dt = _dt(A)
    m = A.shape[1] if trans_a else A.shape[0]
    k = A.shape[0] if trans_a else A.shape[1]
    n = B.shape[0] if trans_b else B.shape[1]
    if C is None:
        C = torch.zeros(m, n, dtype=A.dtype, device=A.device)
    ws = _workspace_named(lib().fb_gemm_workspace_bytes(dt, int(trans_a), int(trans_b), m, n, k), A.device, "gemm", stream)
    _check("fb_gemm", lib().fb_gemm(dt, int(trans_a), int(trans_b), m, n, k, float(alpha), _ptr(A), A.stride(0),
                                    _ptr(B), B.stride(0), float(beta), _ptr(C), C.stride(0), _ptr(ws), ws.numel(),
                                    _stream(stream)))
    return C


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return FB_F32
    if t.dtype == torch.float64:
        return FB_F64
    raise ValueError("fb_matmul supports float32 (3xTF32) and float64 (DMMA)")


def fb_matmul(A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, ws: torch.Tensor | None = None, stream=None):
    m, k = A.shape
    n = B.shape[1]
    _check("fb_matmul", lib().fb_matmul(_dt(A), m, n, k, _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(C),
                                        C.stride(0), _ptr(ws), 0 if ws is None else ws.numel(), _stream(stream)))


def matmul_workspace_bytes(dtype: int, m: int, n: int, k: int) -> int:
    return int(lib().fb_matmul_workspace_bytes(dtype, m, n, k))


def matmul(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """C = A @ B for row-major float32 (3xTF32 tensor cores) or float64 (DMMA) CUDA tensors."""
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0] or A.dtype != B.dtype:
        raise ValueError("shape/dtype mismatch")
    if A.stride(1) != 1 or B.stride(1) != 1:
        raise ValueError("operands must be row-major with unit column stride")
    m, k = A.shape
    n = B.shape[1]
    out = torch.empty((m, n), dtype=A.dtype, device=A.device) if out is None else out
    ws = _workspace(matmul_workspace_bytes(_dt(A), m, n, k), A.device, stream)
    fb_matmul(A, B, out, ws, stream)
    return out


def fb_tf32_split(X: torch.Tensor, hi: torch.Tensor, lo: torch.Tensor, transpose: bool = False, stream=None):
    rows, cols = X.shape
    _check("fb_tf32_split", lib().fb_tf32_split(int(transpose), rows, cols, _ptr(X), X.stride(0), _ptr(hi), _ptr(lo),
                                                hi.stride(0), _stream(stream)))


def fb_matmul_3xtf32_presplit(Ah, Al, Bh, Bl, C, stream=None):
    """C = Ah Bh^T + Ah Bl^T + Al Bh^T  (Ah/Al: m x k, Bh/Bl: n x k, all K-major)."""
    m, k = Ah.shape
    n = Bh.shape[0]
    _check("fb_matmul_3xtf32_presplit", lib().fb_matmul_3xtf32_presplit(
        m, n, k, _ptr(Ah), _ptr(Al), Ah.stride(0), _ptr(Bh), _ptr(Bl), Bh.stride(0), _ptr(C), C.stride(0),
        _stream(stream)))


# ------------------------------------------------------------------ host interface
_named: dict = {}


def _workspace_named(nbytes, device, name, stream=None):
    """Scratch buffer cached per (device, name, stream): calls on different streams never share
    one.  Growing it synchronises the device first, so no kernel queued on that stream still
    uses the old buffer when it goes back to torch's caching allocator."""
    dev = torch.device(device)
    key = (dev.index, name, _stream(stream))
    t = _named.get(key)
    if t is None or t.numel() < nbytes:
        if t is not None:
            torch.cuda.synchronize(dev)
        t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        _named[key] = t
    return t


def fb_fft2d_host(x_host: torch.Tensor, y_host: torch.Tensor, inverse: bool = False, device=0, stream=None):
    """HOST complex64 in -> H2D -> 2D FFT -> D2H -> HOST out (synchronous)."""
    n0, n1 = x_host.shape
    need = lib().fb_fft2d_host_workspace_bytes(n0, n1)
    dev = _workspace_named(need, torch.device("cuda", device), "host_dev", stream)
    _check("fb_fft2d_host", lib().fb_fft2d_host(_ptr(x_host), _ptr(y_host), n0, n1, int(inverse), _ptr(dev),
                                                dev.numel(), _stream(stream)))


def fb_fft2d_host_batch(x_host: torch.Tensor, y_host: torch.Tensor, inverse: bool = False, device=0, stream=None):
    """HOST complex64 [batch, n0, n1] in -> pipelined H2D / 2D FFT / D2H over two device slots
    (copies of consecutive transforms overlap in both PCIe directions) -> HOST out (synchronous)."""
    b, n0, n1 = x_host.shape
    need = lib().fb_fft2d_host_batch_workspace_bytes(n0, n1)
    dev = _workspace_named(need, torch.device("cuda", device), "host_batch_dev", stream)
    _check("fb_fft2d_host_batch", lib().fb_fft2d_host_batch(_ptr(x_host), _ptr(y_host), n0, n1, b, int(inverse),
                                                            _ptr(dev), dev.numel(), _stream(stream)))


def fb_matmul_host(A_host: torch.Tensor, B_host: torch.Tensor, C_host: torch.Tensor, device=0, stream=None):
    m, k = A_host.shape
    n = B_host.shape[1]
    dt = _dt(A_host)
    need = lib().fb_matmul_host_workspace_bytes(dt, m, n, k)
    dev = _workspace_named(need, torch.device("cuda", device), "host_dev", stream)
    _check("fb_matmul_host", lib().fb_matmul_host(dt, m, n, k, _ptr(A_host), _ptr(B_host), _ptr(C_host),
                                                  _ptr(dev), dev.numel(), _stream(stream)))


def fb_lu(A: torch.Tensor, ipiv: torch.Tensor, info: torch.Tensor, stream=None):
    """P A = L U in place (FP64, row-major, LAPACK getrf pivoting; ipiv int32 0-based)."""
    n = A.shape[0]
    _check("fb_lu", lib().fb_lu(FB_F64, n, _ptr(A), A.stride(0), _ptr(ipiv), _ptr(info), None, 0,
                                _stream(stream)))


def lu(A: torch.Tensor, stream=None):
    """Returns (LU, ipiv, info) for a square float64 CUDA tensor (A is not modified)."""
    if A.dtype != torch.float64 or A.dim() != 2 or A.shape[0] != A.shape[1]:
        raise ValueError("lu expects a square float64 CUDA tensor")
    n = A.shape[0]
    ldp = n + (n & 1)  # the C ABI needs an even leading dimension (16-byte rows for DMMA loads)
    buf = torch.zeros(n, ldp, dtype=A.dtype, device=A.device)
    buf[:, :n].copy_(A)
    LU = buf[:, :n]
    ipiv = torch.empty(A.shape[0], dtype=torch.int32, device=A.device)
    info = torch.zeros(1, dtype=torch.int32, device=A.device)
    fb_lu(LU, ipiv, info, stream)
    return LU, ipiv, info


def fb_nr_fourn(data, nn, ndim: int, isign: int):
    """NR fourn(data, nn, ndim, isign) on host numpy arrays with NR's 1-based layout:
    data is float32 of length 2*prod(nn)+1 (data[0] unused), nn is uint64 of length ndim+1."""
    import numpy as np
    if data.dtype != np.float32 or not data.flags.c_contiguous:
        raise ValueError("data must be a contiguous float32 array (NR 1-based)")
    nn = np.ascontiguousarray(nn, dtype=np.uint64)
    _check("fb_nr_fourn", lib().fb_nr_fourn(data.ctypes.data, nn.ctypes.data, ndim, isign))


# ------------------------------------------------------------------ multi-GPU
def slab_rows(rank: int, world: int, n0: int) -> tuple[int, int]:
    """Rows [r0, r1) of the natural n0 x n1 array owned by `rank` (reading R8)."""
    if n0 % world:
        raise ValueError("n0 must be divisible by the world size")
    r = n0 // world
    return rank * r, (rank + 1) * r


def slab_cols(rank: int, world: int, n1: int) -> tuple[int, int]:
    """Columns [c0, c1) of Y held by `rank` after fb_fft2d_slab (reading R8)."""
    if n1 % world:
        raise ValueError("n1 must be divisible by the world size")
    c = n1 // world
    return rank * c, (rank + 1) * c


def exchange_unique_id(rank: int, world: int, make_uid, group=None) -> bytes:
    """Rank 0 creates the communicator id with `make_uid()`; every rank returns the same bytes.
    Uses torch.distributed (any backend) -- plumbing only."""
    raw = make_uid() if rank == 0 else None
    if world > 1:
        import torch.distributed as dist
        obj = [raw]
        dist.broadcast_object_list(obj, src=0, group=group)
        raw = obj[0]
    return bytes(raw)


def _nccl_uid() -> bytes:
    L = lib()
    buf = ctypes.create_string_buffer(L.fb_comm_unique_id_bytes())
    _check("fb_comm_unique_id", L.fb_comm_unique_id(buf))
    return buf.raw


def fb_fft2d_slab_model(P: int, x, y, n0: int, n1: int, inverse: bool = False, stream=None):
    """Single-GPU model of the fused slab path for P virtual ranks (fb.h): forward x (n0 x n1)
    -> y = the P column slabs [P][n0][n1/P]; inverse y -> x."""
    win = torch.empty(n0 * n1, dtype=torch.complex64, device=x.device)
    ws = _workspace_named(lib().fb_fft2d_slab_workspace_bytes(P, n0, n1), x.device, "slab_model", stream)
    _check("fb_fft2d_slab_model", lib().fb_fft2d_slab_model(P, int(inverse), _ptr(x), _ptr(y), n0, n1, _ptr(win),
                                                            _ptr(ws), ws.numel(), _stream(stream)))


class Comm:
    """An fb_comm (NCCL communicator) for this process's GPU."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        raw = exchange_unique_id(rank, world, _nccl_uid, group)
        handle = ctypes.c_void_p()
        _check("fb_comm_init", lib().fb_comm_init(ctypes.byref(handle), world, rank, raw, device))
        self.handle = handle
        self.rank, self.world, self.device = rank, world, device

    @property
    def fused(self) -> bool:
        """True when fb_fft2d_slab moves the column blocks itself over NVLink (fused path)."""
        return bool(lib().fb_comm_fused(self.handle))

    @property
    def fused_detail(self) -> str:
        return lib().fb_comm_fused_detail(self.handle).decode(errors="replace")

    def destroy(self):
        if self.handle:
            _check("fb_comm_destroy", lib().fb_comm_destroy(self.handle))
            self.handle = None

    def fb_fft2d_slab(self, x_rows, y_cols, n0, n1, ws=None, stream=None):
        need = lib().fb_fft2d_slab_workspace_bytes(self.world, n0, n1)
        ws = _workspace_named(need, x_rows.device, "slab", stream) if ws is None else ws
        _check("fb_fft2d_slab", lib().fb_fft2d_slab(self.handle, _ptr(x_rows), _ptr(y_cols), n0, n1, _ptr(ws),
                                                    ws.numel(), _stream(stream)))

    def fb_ifft2d_slab(self, y_cols, x_rows, n0, n1, ws=None, stream=None):
        need = lib().fb_fft2d_slab_workspace_bytes(self.world, n0, n1)
        ws = _workspace_named(need, y_cols.device, "slab", stream) if ws is None else ws
        _check("fb_ifft2d_slab", lib().fb_ifft2d_slab(self.handle, _ptr(y_cols), _ptr(x_rows), n0, n1, _ptr(ws),
                                                      ws.numel(), _stream(stream)))

    def fb_matmul_rowblock(self, A_rows, B, C_rows, root=0, ws=None, stream=None):
        mp, k = A_rows.shape
        n = B.shape[1]
        m = mp * self.world
        dt = _dt(A_rows)
        need = lib().fb_matmul_rowblock_workspace_bytes(self.world, dt, m, n, k)
        ws = _workspace_named(need, A_rows.device, "rowblock", stream) if ws is None else ws
        _check("fb_matmul_rowblock", lib().fb_matmul_rowblock(
            self.handle, dt, m, n, k, _ptr(A_rows), A_rows.stride(0), _ptr(B), B.stride(0), root, _ptr(C_rows),
            C_rows.stride(0), _ptr(ws), ws.numel(), _stream(stream)))
