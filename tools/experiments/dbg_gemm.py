import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb
torch.cuda.set_device(0); fb.fb_init(0)
m = n = 256; k = 64
g = torch.Generator(device="cuda").manual_seed(3)
A = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
B = torch.rand(k, n, device="cuda", generator=g) * 2 - 1
C = fb.matmul(A, B)
torch.cuda.synchronize()
ref = A.double() @ B.double()
err = float(((C.double() - ref).norm() / ref.norm()).item())
A2 = torch.zeros(m, k, device="cuda"); A2[0, 0] = 1.0
B2 = torch.arange(k * n, device="cuda", dtype=torch.float32).reshape(k, n) + 1.0
C2 = fb.matmul(A2, B2); torch.cuda.synchronize()
row = C2[0, :40].cpu().numpy().astype(int).tolist()
print(os.environ.get("TAG", ""), "rel_l2", f"{err:.3e}", "row0", row[:12], row[30:36])
