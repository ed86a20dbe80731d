import os, sys, json, torch
sys.path.insert(0, os.getcwd())
import paper_2004_09883_b200 as fb
torch.cuda.set_device(0); fb.fb_init(0)
for n in (2048, 4096, 8192):
    A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    B = torch.randn(n, n, device="cuda").to(torch.bfloat16)
    C = torch.empty(n, n, device="cuda")
    for bt in (True,):
        for _ in range(3): fb.matmul_bf16(A, B, b_transposed=bt, out=C)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fb.matmul_bf16(A, B, b_transposed=bt, out=C); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = sum(ts) / len(ts)
        ref = None
        for _ in range(3): torch.matmul(A, B)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): torch.matmul(A, B)
        b.record(); torch.cuda.synchronize()
        tc = a.elapsed_time(b) / 10
        print(json.dumps({"n": n, "bt": bt, "ms": t, "tflops": 2 * n**3 / t / 1e9, "cublas_ms": tc, "cublas_tflops": 2 * n**3 / tc / 1e9}))
