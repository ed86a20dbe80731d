"""Context only (never the product path): cuFFT / cuBLAS timings on the same box, same method
(CUDA events, 512 MiB write + 256 MiB read L2 flush before every rep, queue kept ahead)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    evs = []
    for _ in range(reps):
        flush.zero_()
        torch.sum(clean.view(torch.int32))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in evs)
    return ms[len(ms) // 2]


out = {}
for n in (256, 2048, 16384):
    x = torch.randn(n, n, dtype=torch.complex64, device="cuda")
    out[f"cufft_fft2_{n}_ms"] = t(lambda: torch.fft.fft2(x))
    del x
for dt in (torch.float32, torch.float64):
    a = torch.randn(2048, 2048, dtype=dt, device="cuda")
    b = torch.randn(2048, 2048, dtype=dt, device="cuda")
    out[f"cublas_{str(dt)[6:]}_2048_ms"] = t(lambda: a @ b)
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(2048, 2048, device="cuda")
out["cublas_tf32_2048_ms"] = t(lambda: a @ a)
q = torch.randn(2048, 2048, dtype=torch.float64, device="cuda")
out["cusolver_getrf_f64_2048_ms"] = t(lambda: torch.linalg.lu_factor(q))
print(json.dumps(out))
