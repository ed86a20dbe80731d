"""Where the 2048^3 FP32 (3xTF32) fb_matmul call spends its time: whole call, the split pre-pass
pieces and the pre-split tensor-core kernel, each with and without an L2 flush (CUDA events)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = 50
torch.cuda.set_device(0)
fb.fb_init(0)
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
B = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
C = torch.empty(n, n, device="cuda")
ws = torch.empty(fb.matmul_workspace_bytes(fb.FB_F32, n, n, n), dtype=torch.uint8, device="cuda")
Ah, Al, Bh, Bl = (torch.empty(n, n, device="cuda") for _ in range(4))
flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def t(fn, flush):
    ts = []
    for i in range(reps + 5):
        if flush:
            flush_buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return round(ts[len(ts) // 2], 2)


fns = {
    "whole": lambda: fb.fb_matmul(A, B, C, ws, s),
    "split_A_rows": lambda: fb.fb_tf32_split(A, Ah, Al, False, s),
    "split_B_T": lambda: fb.fb_tf32_split(B, Bh, Bl, True, s),
    "presplit_gemm": lambda: fb.fb_matmul_3xtf32_presplit(Ah, Al, Bh, Bl, C, s),
}
out = {"n": n, "env": {k: v for k, v in os.environ.items() if k.startswith("FB_")}}
for k, f in fns.items():
    out[k + "_flush_us"] = t(f, True)
    out[k + "_warm_us"] = t(f, False)
print(json.dumps(out))
