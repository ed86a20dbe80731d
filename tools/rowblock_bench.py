"""fb_matmul_rowblock at world size 1 (real NCCL communicator) vs fb_matmul on the same operands.
usage: python tools/rowblock_bench.py n [reps] [f32|f64]   (knob FB_ROWBLOCK_PANEL = N columns per panel)"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dt = torch.float64 if (len(sys.argv) > 3 and sys.argv[3] == "f64") else torch.float32
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
fb.fb_init(0)
comm = fb.Comm(0, 1, 0)
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(dt)
B = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(dt)
C1 = torch.empty(n, n, device="cuda", dtype=dt)
C2 = torch.empty_like(C1)
s = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sum(ts) / len(ts)


t_mm = timed(lambda: fb.matmul(A, B, out=C1))
t_rb = timed(lambda: comm.fb_matmul_rowblock(A, B, C2, root=0))
print(json.dumps({"n": n, "dtype": str(dt), "fb_matmul_ms": t_mm, "rowblock_ms": t_rb, "ratio": t_rb / t_mm,
                  "bitwise_equal": bool(torch.equal(C1, C2)), "panel": os.environ.get("FB_ROWBLOCK_PANEL", "4096")}))
comm.destroy()
dist.destroy_process_group()
