"""Per-configuration timing of fb_fft2d (CUDA events, L2 flushed) for A/B tuning runs.

usage: python tools/fft_pass_bench.py n0 n1 [reps]   (env knobs: FB_FFT_* in csrc/fb_fft.cu)
Prints one JSON line {n0, n1, ms, ms_min, knobs}.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

n0, n1 = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
torch.cuda.set_device(0)
fb.fb_init(0)
x = (torch.randn(n0, n1, dtype=torch.complex64, device="cuda"))
y = torch.empty_like(x)
ws_b = fb.lib().fb_fft2d_workspace_bytes(n0, n1)
ws = torch.empty(max(ws_b, 1), dtype=torch.uint8, device="cuda") if ws_b else None
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
mode = os.environ.get("FLUSH", "write")  # none | write | write+read


def do_flush():
    if mode == "none":
        return
    flush.zero_()
    if mode == "write+read":
        clean.sum()
s = torch.cuda.current_stream()
ts = []
for i in range(reps + 5):
    do_flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fb.fb_fft2d(x, y, ws, s)
    b.record(s)
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(a.elapsed_time(b))
ts.sort()
knobs = {k: v for k, v in os.environ.items() if k.startswith("FB_FFT") or k == "FLUSH"}
print(json.dumps({"n0": n0, "n1": n1, "ms": sum(ts) / len(ts), "ms_min": ts[0], "ms_med": ts[len(ts) // 2],
                  "ms_p10": ts[len(ts) // 10], "ms_p90": ts[(9 * len(ts)) // 10],
                  "knobs": knobs}))
