"""How does tcgen05 kind::tf32 read an FP32 operand whose low 13 mantissa bits are NOT zero?
(truncate, round-to-nearest, or use them).  C = Ah Bh^T with Al = Bl = 0, Bh = e_0 (one 1.0):
C[i][0] = hw(Ah[i][0]).  Prints the fraction of rows matching each rule."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

torch.cuda.set_device(0)
fb.fb_init(0)
m, n, k = 256, 256, 32
rng = np.random.default_rng(1)
a = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
a[:, 0] = (rng.uniform(1, 2, size=m) * np.sign(rng.uniform(-1, 1, size=m))).astype(np.float32)
A = torch.from_numpy(a).cuda()
Z = torch.zeros_like(A)
B = torch.zeros(n, k, device="cuda")
B[0, 0] = 1.0
C = torch.empty(m, n, device="cuda")
fb.fb_matmul_3xtf32_presplit(A, Z, B, torch.zeros_like(B), C)
torch.cuda.synchronize()
c = C[:, 0].cpu().numpy()
x = a[:, 0]
bits = x.view(np.uint32)
trunc = (bits & np.uint32(0xFFFFE000)).view(np.float32)
# round to nearest even at bit 13
lsb = (bits >> np.uint32(13)) & np.uint32(1)
rne = ((bits + np.uint32(0x0FFF) + lsb) & np.uint32(0xFFFFE000)).view(np.float32)
rna = ((bits + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)
print({"exact_fp32": float(np.mean(c == x)), "trunc": float(np.mean(c == trunc)), "rne": float(np.mean(c == rne)),
       "rna": float(np.mean(c == rna)), "rows": m})
