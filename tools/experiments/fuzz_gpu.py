"""Randomised shape fuzzing of the GPU paths (not a test; a bug hunt): 2D FFT of random
power-of-two / 7-smooth / other sizes (forward vs numpy.fft in FP64, round trip), fb_gemm with
random m, n, k, transposes, alpha/beta (vs torch FP64), BF16 GEMM.  Prints failures and a summary.
usage: python tools/experiments/fuzz_gpu.py [n_cases] [seed]"""
import os
import random
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2004_09883_b200 as fb  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
torch.cuda.set_device(0)
fb.fb_init(0)
fails = []
counts = {"fft2d": 0, "gemm": 0, "bf16": 0, "fft1d": 0, "rfft2d": 0, "slab": 0}


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def fft_size():
    r = rng.random()
    if r < 0.4:
        return 2 ** rng.randint(0, 14)
    if r < 0.75:
        while True:
            n = (2 ** rng.randint(0, 6)) * (3 ** rng.randint(0, 4)) * (5 ** rng.randint(0, 3)) * (7 ** rng.randint(0, 2))
            if n <= 4096:
                return n
    return rng.randint(1, 3000)


for case in range(N):
    kind = rng.random()
    try:
        if kind < 0.45:
            n0, n1 = fft_size(), fft_size()
            if n0 * n1 > (1 << 24):
                continue
            x = (np.random.default_rng(case).standard_normal((n0, n1)) +
                 1j * np.random.default_rng(case + 1).standard_normal((n0, n1))).astype(np.complex64)
            xd = torch.from_numpy(x).cuda()
            y = fb.fft2d(xd).cpu().numpy()
            z = fb.fft2d(torch.from_numpy(y).cuda(), inverse=True).cpu().numpy()
            ref = np.fft.fft2(x.astype(np.complex128))
            e, ei = rel(y, ref), rel(z, x)
            bar = 1e-5 * max(1.0, np.log2(n0 * n1))
            counts["fft2d"] += 1
            if not (e < bar and ei < bar):
                fails.append(("fft2d", n0, n1, e, ei))
        elif kind < 0.85:
            dt = torch.float32 if rng.random() < 0.6 else torch.float64
            q = 4 if dt == torch.float32 else 2
            m = rng.randint(1, 1500)
            n = rng.randint(1, 1500) // q * q or q
            k = rng.randint(1, 1500) // q * q or q
            ta, tb = rng.random() < 0.3, rng.random() < 0.3
            if ta and m % q:
                m = (m // q + 1) * q
            alpha, beta = rng.choice([(1.0, 0.0), (0.5, -1.5), (2.0, 1.0), (0.0, 0.5)])
            g = torch.Generator(device="cuda").manual_seed(case)
            A = torch.rand((k, m) if ta else (m, k), device="cuda", generator=g, dtype=torch.float64) * 2 - 1
            B = torch.rand((n, k) if tb else (k, n), device="cuda", generator=g, dtype=torch.float64) * 2 - 1
            C0 = torch.rand((m, n), device="cuda", generator=g, dtype=torch.float64) * 2 - 1
            C = C0.to(dt).clone()
            fb.gemm(A.to(dt), B.to(dt), C, alpha, beta, ta, tb)
            opA = (A.to(dt).double().t() if ta else A.to(dt).double())
            opB = (B.to(dt).double().t() if tb else B.to(dt).double())
            ref = alpha * (opA @ opB) + beta * C0.to(dt).double()
            e = rel(C.double().cpu().numpy(), ref.cpu().numpy())
            counts["gemm"] += 1
            if not e < (1e-5 if dt == torch.float32 else 1e-12):
                fails.append(("gemm", str(dt), m, n, k, ta, tb, alpha, beta, e))
        elif kind < 0.90:
            sub = rng.random()
            if sub < 0.4:  # batched 1D
                n, b = 2 ** rng.randint(0, 14), rng.randint(1, 300)
                x = (np.random.default_rng(case).standard_normal((b, n)) +
                     1j * np.random.default_rng(case + 2).standard_normal((b, n))).astype(np.complex64)
                y = fb.fft1d(torch.from_numpy(x).cuda()).cpu().numpy()
                e = rel(y, np.fft.fft(x.astype(np.complex128), axis=1))
                counts["fft1d"] += 1
                if not e < 1e-5 * max(1.0, np.log2(n)):
                    fails.append(("fft1d", b, n, e))
            elif sub < 0.7:  # real input
                n0, n1 = 2 ** rng.randint(0, 11), 2 ** rng.randint(1, 11)
                x = np.random.default_rng(case).standard_normal((n0, n1)).astype(np.float32)
                y = fb.rfft2d(torch.from_numpy(x).cuda())
                z = fb.irfft2d(y, n1).cpu().numpy()
                e, ei = rel(y.cpu().numpy(), np.fft.rfft2(x.astype(np.float64))), rel(z, x)
                counts["rfft2d"] += 1
                if not (e < 1e-5 * max(1.0, np.log2(n0 * n1)) and ei < 1e-5 * max(1.0, np.log2(n0 * n1))):
                    fails.append(("rfft2d", n0, n1, e, ei))
            else:  # slab model, P virtual ranks
                P = rng.choice([1, 2, 4, 8])
                n0, n1 = 2 ** rng.randint(3, 12), 2 ** rng.randint(3, 12)
                x = (np.random.default_rng(case).standard_normal((n0, n1)) +
                     1j * np.random.default_rng(case + 3).standard_normal((n0, n1))).astype(np.complex64)
                xd = torch.from_numpy(x).cuda()
                yd = torch.empty(n0 * n1, dtype=torch.complex64, device="cuda")
                fb.fb_fft2d_slab_model(P, xd, yd, n0, n1)
                y = yd.view(P, n0, n1 // P).permute(1, 0, 2).reshape(n0, n1).cpu().numpy()
                e = rel(y, np.fft.fft2(x.astype(np.complex128)))
                counts["slab"] += 1
                if not e < 1e-5 * max(1.0, np.log2(n0 * n1)):
                    fails.append(("slab", P, n0, n1, e))
        else:
            m = rng.randint(1, 1200)
            n = rng.randint(1, 1200) // 8 * 8 or 8
            k = rng.randint(1, 1200) // 8 * 8 or 8
            bt = rng.random() < 0.5
            g = torch.Generator(device="cuda").manual_seed(case)
            A = (torch.rand(m, k, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            Bk = (torch.rand(k, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
            C = fb.matmul_bf16(A, Bk.t().contiguous() if bt else Bk, b_transposed=bt)
            ref = A.double() @ Bk.double()
            e = rel(C.double().cpu().numpy(), ref.cpu().numpy())
            counts["bf16"] += 1
            if not e < 1e-5:
                fails.append(("bf16", m, n, k, bt, e))
    except Exception as ex:  # noqa: BLE001
        fails.append(("exception", case, repr(ex)[:200]))
torch.cuda.synchronize()
print(f"{N} cases {counts}, {len(fails)} failures")
for f in fails[:40]:
    print(f)
