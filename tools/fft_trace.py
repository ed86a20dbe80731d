"""Per-CTA timeline of the two 2048^2 pair-plan passes (trace build of libfb: -DFB_FFT_TRACE=1).

usage: FB_LIB=paper_2004_09883_b200/libfb_trace.so python tools/fft_trace.py [n] [stagger...]
Prints, per pass: launch-to-start spread, per-group wait (mbarrier) and compute times, the
exit-time distribution and the gap between the passes (globaltimer, ns).
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2004_09883_b200 as fb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
torch.cuda.set_device(0)
fb.fb_init(0)
L = fb.lib()
buf = torch.zeros(2 * 1024 * 32, dtype=torch.int64, device="cuda")
L.fb_debug_fft_trace.argtypes = [ctypes.c_void_p]
x = torch.randn(n, n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
ws = torch.empty(L.fb_fft2d_workspace_bytes(n, n), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(256 << 20, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
res = []
for rep in range(8):
    flush.zero_()
    clean.sum()
    buf.zero_()
    torch.cuda.synchronize()
    L.fb_debug_fft_trace(ctypes.c_void_p(buf.data_ptr()))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fb.fb_fft2d(x, y, ws, s)
    b.record(s)
    torch.cuda.synchronize()
    L.fb_debug_fft_trace(ctypes.c_void_p(0))
    t = buf.view(2, 1024, 32).cpu().numpy().astype(np.int64)
    res.append((a.elapsed_time(b) * 1e3, t))
ev_us, t = res[-1]
out = {"n": n, "event_us": ev_us}
t0 = None
prev_exit = None
for slot, name in ((0, "row"), (1, "col")):
    tt = t[slot]
    used = tt[:, 1] > 0
    tt = tt[used]
    if not len(tt):
        continue
    if t0 is None:
        t0 = tt[:, 1].min()
    ng = tt[:, 31]
    start = (tt[:, 1] - t0) / 1e3
    exit_ = (tt[:, 30] - t0) / 1e3
    waits, comps, first_wait = [], [], []
    for r in tt:
        g = int(r[31])
        for i in range(min(g, 14)):
            top, ready = r[2 + 2 * i], r[3 + 2 * i]
            w = (ready - top) / 1e3
            (first_wait if i == 0 else waits).append(w)
            end = r[2 + 2 * (i + 1)] if i + 1 < min(g, 14) else r[30]
            comps.append((end - ready) / 1e3)
    d = {"ctas": int(used.sum()), "groups_per_cta": np.bincount(ng).tolist(),
         "start_us": [round(float(np.min(start)), 2), round(float(np.median(start)), 2), round(float(np.max(start)), 2)],
         "exit_us": [round(float(np.min(exit_)), 2), round(float(np.percentile(exit_, 10)), 2),
                     round(float(np.median(exit_)), 2), round(float(np.percentile(exit_, 90)), 2),
                     round(float(np.max(exit_)), 2)],
         "first_wait_us": [round(float(np.min(first_wait)), 2), round(float(np.median(first_wait)), 2),
                           round(float(np.max(first_wait)), 2)],
         "later_wait_us_mean": round(float(np.mean(waits)), 3) if waits else None,
         "compute_us": [round(float(np.min(comps)), 2), round(float(np.median(comps)), 2), round(float(np.max(comps)), 2)]}
    # exit time by number of groups
    d["exit_by_groups"] = {int(k): round(float(np.median(exit_[ng == k])), 2) for k in np.unique(ng)}
    # per SM: groups, first start, last exit (sorted by last exit)
    sm = {}
    for r, st_, ex in zip(tt, start, exit_):
        e = sm.setdefault(int(r[0]), [0, 1e9, 0.0, 0])
        e[0] += int(r[31]); e[1] = min(e[1], st_); e[2] = max(e[2], ex); e[3] += 1
    rows_ = sorted(sm.items(), key=lambda kv: kv[1][2])
    d["sm_count"] = len(rows_)
    d["sm_groups_hist"] = np.bincount([v[0] for _, v in rows_]).tolist()
    d["sm_last_exit_us"] = [round(float(np.percentile([v[2] for _, v in rows_], q)), 2) for q in (0, 10, 50, 90, 100)]
    d["sm_fastest"] = [(k, v[0], round(v[2], 2)) for k, v in rows_[:4]]
    d["sm_slowest"] = [(k, v[0], round(v[2], 2)) for k, v in rows_[-4:]]
    if os.environ.get("TRACE_SM"):
        for smid in [rows_[0][0], rows_[len(rows_) // 2][0], rows_[-1][0]]:
            for r in tt[tt[:, 0] == smid]:
                g = int(r[31])
                ev = [round((r[1] - t0) / 1e3, 2)] + [(round((r[2 + 2 * i] - t0) / 1e3, 2), round((r[3 + 2 * i] - t0) / 1e3, 2)) for i in range(min(g, 14))] + [round((r[30] - t0) / 1e3, 2)]
                print(name, "sm", smid, "groups", g, ev)
    if prev_exit is not None:
        d["gap_after_prev_pass_us"] = round(float(np.min(start) - prev_exit), 2)
    prev_exit = float(np.max(exit_))
    out[name] = d
print(json.dumps(out))
