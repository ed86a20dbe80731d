"""Small invocations of every kernel family, for compute-sanitizer (racecheck / synccheck /
memcheck, one tool per run): FFT 256^2, 2048 x 64, 64 x 2048 (TMA row/column passes, pair plan,
sub-CTA pass), GEMM 512^3 FP32 (split + CTA-pair tcgen05, fused variant) and FP64 (DMMA), LU 192."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

torch.cuda.set_device(0)
fb.fb_init(0)
g = torch.Generator(device="cuda").manual_seed(0)
for n0, n1 in ((256, 256), (2048, 64), (64, 2048), (512, 512)):
    x = torch.randn(n0, n1, dtype=torch.complex64, device="cuda", generator=g)
    y = fb.fft2d(x)
    z = fb.ifft2d(y)
A = torch.rand(512, 512, device="cuda", generator=g)
B = torch.rand(512, 512, device="cuda", generator=g)
C = fb.matmul(A, B)
C64 = fb.matmul(A.double(), B.double())
if os.environ.get("SAN_FUSED", "1") == "1":
    os.environ["FB_GEMM_FUSED"] = "1"
    fb.fb_reload_knobs()
    Cf = fb.matmul(A, B)
    os.environ["FB_GEMM_FUSED"] = "0"
    fb.fb_reload_knobs()
M = torch.rand(192, 192, device="cuda", dtype=torch.float64, generator=g)
ipiv = torch.empty(192, dtype=torch.int32, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
fb.fb_lu(M, ipiv, info)
torch.cuda.synchronize()
print("sanitize target done")
