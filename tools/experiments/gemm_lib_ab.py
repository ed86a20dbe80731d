"""fb_matmul FP32 timing through a given libfb build (raw ctypes, no binding), L2 flushed.
usage: python tools/experiments/gemm_lib_ab.py LIB.so n [reps]"""
import ctypes
import json
import sys

import torch

lib = ctypes.CDLL(sys.argv[1])
n = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
vp, i64, sz, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
lib.fb_init.argtypes = [ci]
lib.fb_matmul_workspace_bytes.argtypes = [ci, i64, i64, i64]
lib.fb_matmul_workspace_bytes.restype = sz
lib.fb_matmul.argtypes = [ci, i64, i64, i64, vp, i64, vp, i64, vp, i64, vp, sz, vp]
torch.cuda.set_device(0)
assert lib.fb_init(0) == 0
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
B = torch.rand(n, n, device="cuda", generator=g) * 2 - 1
C = torch.empty(n, n, device="cuda")
wsb = lib.fb_matmul_workspace_bytes(0, n, n, n)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
ts = []
for i in range(reps + 3):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    assert lib.fb_matmul(0, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, ws.data_ptr(), wsb,
                         s.cuda_stream) == 0
    b.record(s)
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b))
print(json.dumps({"lib": sys.argv[1].split("/")[-1], "n": n, "us": 1e3 * sum(ts) / len(ts)}))
