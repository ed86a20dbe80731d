"""Timing of fb_matmul (CUDA events, L2 flushed before each rep) for A/B runs.
usage: python tools/gemm_bench.py m n k [reps] [f32|f64]   (env knobs FB_GEMM_*)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

m, n, k = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
dt = torch.float64 if (len(sys.argv) > 5 and sys.argv[5] == "f64") else torch.float32
torch.cuda.set_device(0)
fb.fb_init(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(dt)
B = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1).to(dt)
C = torch.empty(m, n, device="cuda", dtype=dt)
ws = torch.empty(max(1, fb.matmul_workspace_bytes(fb.FB_F32 if dt == torch.float32 else fb.FB_F64, m, n, k)),
                 dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
ts = []
for i in range(reps + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fb.fb_matmul(A, B, C, ws, s)
    b.record(s)
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
ref = (A.double() @ B.double())
err = float(((C.double() - ref).norm() / ref.norm()).item())
t = sum(ts) / len(ts)
print(json.dumps({"m": m, "n": n, "k": k, "dtype": str(dt), "ms": t, "ms_min": min(ts),
                  "tflops": 2.0 * m * n * k / (t * 1e-3) / 1e12, "rel_l2_vs_torch_f64": err,
                  "knobs": {kk: v for kk, v in os.environ.items() if kk.startswith("FB_GEMM")}}))
