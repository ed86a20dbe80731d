import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2004_09883_b200 as fb, oracle, synth
torch.cuda.set_device(0); fb.fb_init(0)
for n in [24, 33]:
    A = synth.real_matrix(n, n, synth.TID_GEMM_A).astype(np.float64)
    res = {}
    for knob in ["1", "0"]:
        os.environ["FB_LU_TMA"] = knob
        LU, piv, info = fb.lu(torch.from_numpy(A).cuda())
        torch.cuda.synchronize()
        res[knob] = (LU.cpu().numpy(), piv.cpu().numpy(), info)
    print(n, "ipiv tma ", res["1"][1].tolist())
    print(n, "ipiv cpas", res["0"][1].tolist())
    d = np.abs(res["1"][0] - res["0"][0])
    np.set_printoptions(linewidth=250, precision=2)
    print((d > 1e-9).astype(int))
