"""BF16 GEMM timing at given sizes (CUDA events, L2 flushed before each rep), for A/B runs.
usage: python tools/experiments/bf16_size_bench.py n [reps]   (env knobs FB_BF16_*)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2004_09883_b200 as fb  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
torch.cuda.set_device(0)
fb.fb_init(0)
g = torch.Generator(device="cuda").manual_seed(5)
A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
Bt = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
C = torch.empty(n, n, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(reps + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fb.matmul_bf16(A, Bt, b_transposed=True, out=C)
    b.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
t = sum(ts) / len(ts)
print(json.dumps({"n": n, "ms": t, "tflops": 2 * n ** 3 / (t * 1e-3) / 1e12,
                  "knobs": {k: v for k, v in os.environ.items() if k.startswith("FB_BF16")}}))
