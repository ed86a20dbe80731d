"""Time fb_fft2d_slab / fb_ifft2d_slab at world size 1 (fused transpose vs NCCL all-to-all path;
FB_SLAB_FUSED=0 selects the latter).  usage: python tools/slab_bench.py n0 n1 [reps]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

n0, n1 = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
torch.cuda.set_device(0)
fb.fb_init(0)
comm = fb.Comm(0, 1, 0)
x = torch.randn(n0, n1, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
z = torch.empty_like(x)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
res = {}
for name, fn in [("fwd", lambda: comm.fb_fft2d_slab(x, y, n0, n1)), ("inv", lambda: comm.fb_ifft2d_slab(y, z, n0, n1))]:
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    res[name] = sum(ts) / len(ts)
print(json.dumps({"n0": n0, "n1": n1, "fused": comm.fused, "ms": res}))
comm.destroy()
