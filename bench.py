#!/usr/bin/env python
"""bench.py -- throughput of the function blocks of arXiv 2004.09883 on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fb|reference] [--workload W]

One JSON line on rank 0.  Headline workload (N=1): BASELINE configs[1], the paper-shaped
Fourier-transform block: a forward complex 2D FFT of one 2048x2048 complex64 batch
("grid size 2048*2048").  The matrix block (configs[2], 2048^3 GEMM in FP32
3xTF32 and FP64) is measured in the same run and reported under "blocks" with its own
roofline; so are the 256^2 forward+inverse (configs[0]) and the single-GPU 16384^2 FFT
(the scaling baseline for configs[3]).  With N>1 ranks (torchrun) the headline is
configs[3]: the slab-sharded 16384^2 FFT with its NCCL all-to-all (strong scaling).

Timing: inputs resident in HBM; before every timed step L2 is flushed by a 512 MiB memset
followed by a 1 GiB read (untimed; leaves L2 clean); each step is bracketed by CUDA events on the launching stream; barrier +
synchronize around the timed region; max over ranks.  FLOP conventions: FFT 5 N log2 N
(N = n0 n1), GEMM 2 M N K.  The `--impl reference` arm times the CPU oracle (oracle/) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D FFT GFLOP/s & GEMM TFLOP/s at 1/2/4/8 B200; % of HBM/TC roofline"
FLUSH_BYTES = 512 << 20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


def tc_peaks():
    """tensor-core peaks measured on this pool's B200 by tools/peak_tc.cu
    (profiles/r2_peaks.json): TF32 tcgen05 burst / sustained (data operands; the sustained run
    sits at the 1 kW power cap) and FP64 DMMA.  One derivation for every GEMM roofline."""
    p = os.path.join(ROOT, "profiles", "r2_peaks.json")
    d = json.load(open(p))
    return {"tf32_burst": float(d["tf32"]["use"]["burst"]), "tf32_sustained": float(d["tf32"]["use"]["sustained"]),
            "f64": float(d["fp64_dmma"]["use"]),
            "source": "measured: profiles/r2_peaks.json (tools/peak_tc.cu tcgen05 kind::tf32 / DMMA issue loops)"}


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def ncu_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the workload's dominant kernel(s),
    from the committed `ncu --set full` summaries (profiles/ncu_traffic.json, written by
    tools/ncu_summarize.py), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    vals = list(json.load(open(p)).get(workload, {}).values())
    return float(vals[0]) if vals else None


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- timing helpers
def timed_steps(torch, fn, steps, warmup, flush, stream, dist=None):
    """W untimed warm-ups, then exactly K steps; per-step CUDA events on `stream`, L2 flushed
    (untimed) before each.  Returns per-step ms list (max over ranks of the mean applied by caller)."""
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            flush()
            fn()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            flush()
            a.record(stream)
            fn()
            b.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def max_over_ranks(torch, dist, v):
    if dist is None:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def fft_flops(n0, n1):
    n = n0 * n1
    return 5.0 * n * math.log2(n) if n > 1 else 0.0


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm (no GPU work)."""
    import numpy as np

    import oracle
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n = 2048
    x = synth.complex_field(n, n)
    cols_per_step = 16
    threads = oracle.threads(0)
    flop_equiv = fft_flops(n, n) * cols_per_step / n

    def step(i):
        for j in range(cols_per_step):
            oracle.dft2d_col(x, (i * cols_per_step + j) % n)

    for i in range(args.warmup):
        step(i)
    ts = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        step(i)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(ts))
    val = flop_equiv / (ms * 1e-3) / 1e9
    sample = (f"{cols_per_step} full output columns of the 2048x2048 forward 2D DFT per step "
              f"(naive O(n^2) definition, FP64), scaled to the 5 N log2 N flop count of the full transform")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.gpus > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "fft2d_2048x2048_fwd", "n0": n, "n1": n},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- fb arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fb", choices=["fb", "reference"])
    ap.add_argument("--no-extras", action="store_true", help="headline only (no blocks / cpu baseline / e2e)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--only", default="", help="comma list of blocks to run (debug)")
    ap.add_argument("--slab", action="store_true",
                    help="run the multi-GPU headline (slab-sharded 16384^2) even at world size 1 (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    import paper_2004_09883_b200 as fb
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fb.fb_init(local)
    stream = torch.cuda.Stream()
    pk = peaks()
    flush_buf = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
    clean_buf = torch.ones(FLUSH_BYTES // 2, dtype=torch.float32, device="cuda")  # 1 GiB

    def flush():
        # write 512 MiB (> 126 MB L2) then read 1 GiB so that L2 holds only clean lines:
        # the flush's own dirty lines are not written back inside the next timed step
        flush_buf.zero_()
        clean_buf.sum()  # float32 reduction: reads only, no dtype-promotion copy

    only = set(filter(None, args.only.split(",")))
    out = {"metric": METRIC, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "higher_is_better": True, "vs_baseline": None, "dtype": "f32", "data": "synthetic"}
    blocks = {}

    # ------------------------------------------------------------------ N = 1 headline: 2048^2 FFT
    if world == 1 and not args.slab:
        n = 2048
        x_h = synth.complex_field(n, n)
        x = torch.from_numpy(x_h).cuda()
        y = torch.empty_like(x)
        wsb = fb.lib().fb_fft2d_workspace_bytes(n, n)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda") if wsb else None
        L0 = fb.launch_count()
        with ClockSampler(local) as clk:
            ms = timed_steps(torch, lambda: fb.fb_fft2d(x, y, ws, stream), args.steps, args.warmup, flush, stream)
        launches = (fb.launch_count() - L0) // (args.steps + args.warmup)
        t = float(np.mean(ms))
        gflops = fft_flops(n, n) / (t * 1e-3) / 1e9
        # the FFT pass kernels (2 launches per step: the radix-16 pair row pass
        # fft_pass_tma_kernel and the radix-32 column pass fft_col1024_kernel); each launch reads
        # and writes the 32 MiB array once -> 64 MiB algorithmic bytes per launch.
        bytes_launch = 2 * 8 * n * n
        achieved = bytes_launch / ((t / launches) * 1e-3) / 1e9
        out.update({"value": gflops, "unit": "GFLOP/s", "ms_per_step": t, "scaling": "strong",
                    "config": {"workload": "fft2d_2048x2048_fwd", "n0": n, "n1": n, "element": "complex64",
                               "l2": "flushed before every timed step (untimed): 512 MiB memset + 1 GiB read",
                               "configs_index": 1},
                    "roofline": {"bound": "hbm",
                                 "kernel": "fft_pass_tma_kernel (row pass) + fft_col1024_kernel (column pass)",
                                 "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                 "frac": achieved / pk["hbm_gbs"],
                                 "traffic": ncu_traffic("fft2d_2048"),
                                 "algorithmic_bytes_per_launch": bytes_launch,
                                 "launches_per_step": launches, "peak_source": pk["source"]},
                    "gpu_launches": launches * args.steps, "clocks": clk.summary()})

        # e2e through the public host API: pinned host in -> H2D -> FFT -> D2H -> pinned host out.
        # Headline: the streaming host call (E2E_BATCH transforms per call, two device slots so
        # transform i+1's H2D overlaps transform i's D2H); the one-transform synchronous call is
        # reported beside it.
        if not args.no_extras:
            E2E_BATCH = 8

            def host_timed(call, reps):
                ets = []
                for _ in range(reps):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(stream):
                        flush()
                    torch.cuda.synchronize()
                    a.record(stream)
                    call()
                    b.record(stream)
                    torch.cuda.synchronize()
                    ets.append(a.elapsed_time(b))
                return float(np.mean(ets))

            xh = torch.from_numpy(x_h).pin_memory()
            yh = torch.empty_like(xh).pin_memory()
            xb = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(x_h, (E2E_BATCH,) + x_h.shape))).pin_memory()
            yb = torch.empty_like(xb).pin_memory()
            for _ in range(args.warmup):
                fb.fb_fft2d_host(xh, yh, stream=stream)
                fb.fb_fft2d_host_batch(xb, yb, stream=stream)
            te1 = host_timed(lambda: fb.fb_fft2d_host(xh, yh, stream=stream), args.steps)
            teb = host_timed(lambda: fb.fb_fft2d_host_batch(xb, yb, stream=stream), args.steps)
            assert np.array_equal(yb[E2E_BATCH - 1].numpy().view(np.uint32), yh.numpy().view(np.uint32))
            out["e2e"] = {"value": E2E_BATCH * fft_flops(n, n) / (teb * 1e-3) / 1e9, "unit": "GFLOP/s",
                          "ms_per_step": teb, "transforms_per_step": E2E_BATCH,
                          "h2d_bytes_per_step": int(xb.numel() * 8), "d2h_bytes_per_step": int(yb.numel() * 8),
                          "api": "fb_fft2d_host_batch (pinned host buffers; two device slots, copies of "
                                 "consecutive transforms overlap in both PCIe directions)",
                          "single_call": {"value": fft_flops(n, n) / (te1 * 1e-3) / 1e9, "unit": "GFLOP/s",
                                          "ms_per_step": te1, "h2d_bytes_per_step": int(xh.numel() * 8),
                                          "d2h_bytes_per_step": int(yh.numel() * 8),
                                          "api": "fb_fft2d_host (one transform, synchronous)"}}

        # CPU oracle baseline on the same input: the full 2048^2 definition (~10-30 s)
        if not (args.no_extras or args.no_cpu_baseline):
            import oracle
            thr = oracle.threads(0)
            t0 = time.perf_counter()
            ref = oracle.dft2d(x_h, nthreads=thr)
            tcpu = time.perf_counter() - t0
            err = oracle.rel_l2(y.cpu().numpy(), ref)
            out["cpu_baseline"] = {"value": fft_flops(n, n) / tcpu / 1e9, "unit": "GFLOP/s", "cores": thr,
                                   "kind": "oracle", "seconds": tcpu, "cpu": cpu_model(),
                                   "sample": "the full 2048x2048 forward 2D DFT (naive O(n^2) per line, FP64) "
                                             "on the bench input, flops counted as 5 N log2 N"}
            out["parity"] = {"fft2d_2048_rel_l2_vs_oracle": err, "bar": 1e-5 * math.log2(n * n)}

        if not args.no_extras:
            blocks.update(extra_blocks(args, torch, fb, synth, np, stream, flush, pk, only))
    else:
        out.update(run_slab(args, torch, fb, synth, np, stream, flush, pk, dist, rank, world, local))

    if blocks:
        out["blocks"] = blocks
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def extra_blocks(args, torch, fb, synth, np, stream, flush, pk, only):
    res = {}
    steps = max(3, args.steps // 2)

    def want(k):
        return not only or k in only

    # configs[2]: GEMM 2048^3 FP32 (3xTF32 tcgen05) and FP64 (DMMA)
    n = 2048
    if want("gemm_f32_2048"):
        A = torch.from_numpy(synth.real_matrix(n, n, synth.TID_GEMM_A)).cuda()
        B = torch.from_numpy(synth.real_matrix(n, n, synth.TID_GEMM_B)).cuda()
        C = torch.empty(n, n, device="cuda")
        ws = torch.empty(fb.matmul_workspace_bytes(fb.FB_F32, n, n, n), dtype=torch.uint8, device="cuda")
        ms = timed_steps(torch, lambda: fb.fb_matmul(A, B, C, ws, stream), steps, args.warmup, flush, stream)
        t = float(np.mean(ms))
        # the tensor-core kernel alone (operands pre-split)
        kp = (n + 3) // 4 * 4
        Ah = torch.empty(n, kp, device="cuda")
        Al = torch.empty_like(Ah)
        Bh = torch.empty(n, kp, device="cuda")
        Bl = torch.empty_like(Bh)
        fb.fb_tf32_split(A, Ah, Al, False, stream)
        fb.fb_tf32_split(B, Bh, Bl, True, stream)
        mk = timed_steps(torch, lambda: fb.fb_matmul_3xtf32_presplit(Ah, Al, Bh, Bl, C, stream), steps,
                         args.warmup, flush, stream)
        tk = float(np.mean(mk))
        flops = 2.0 * n * n * n
        tcp = tc_peaks()
        tf32_peak = tcp["tf32_burst"]  # measured tcgen05 kind::tf32 burst peak (K8)
        res["gemm_f32_2048"] = {
            "value": flops / (t * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": t,
            "config": {"workload": "gemm_2048^3_fp32_3xtf32", "configs_index": 2},
            "roofline": {"bound": "tensor", "kernel": "gemm_3xtf32_kernel", "kernel_ms": tk,
                         "achieved": 3 * flops / (tk * 1e-3) / 1e12, "peak": tf32_peak, "unit": "TFLOP/s",
                         "frac": 3 * flops / (tk * 1e-3) / 1e12 / tf32_peak,
                         "note": "achieved counts the 3 TF32 MMAs (6MNK); useful 2MNK = achieved/3",
                         "traffic": ncu_traffic("gemm_2048"),
                         "whole_call_frac": 3 * flops / (t * 1e-3) / 1e12 / tf32_peak,
                         "peak_source": tcp["source"] + " -- TF32 burst, data operands"}}
        del A, B, C, ws, Ah, Al, Bh, Bl
    if want("gemm_f64_2048"):
        A = torch.from_numpy(synth.real_matrix(n, n, synth.TID_GEMM_A, dtype=np.float64)).cuda()
        B = torch.from_numpy(synth.real_matrix(n, n, synth.TID_GEMM_B, dtype=np.float64)).cuda()
        C = torch.empty(n, n, device="cuda", dtype=torch.float64)
        ms = timed_steps(torch, lambda: fb.fb_matmul(A, B, C, None, stream), steps, args.warmup, flush, stream)
        t = float(np.mean(ms))
        flops = 2.0 * n * n * n
        f64_peak = tc_peaks()["f64"]  # measured DMMA peak (K8)
        res["gemm_f64_2048"] = {
            "value": flops / (t * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": t,
            "config": {"workload": "gemm_2048^3_fp64_dmma", "configs_index": 2},
            "roofline": {"bound": "tensor", "kernel": "gemm_f64_dmma_kernel", "achieved": flops / (t * 1e-3) / 1e12,
                         "peak": f64_peak, "unit": "TFLOP/s", "frac": flops / (t * 1e-3) / 1e12 / f64_peak,
                         "traffic": ncu_traffic("gemm_f64_2048"),
                         "peak_source": tc_peaks()["source"] + " -- FP64 DMMA"}}
        del A, B, C
    # the paper's own matrix workload, LU of a 2048x2048 orthogonal matrix
    if want("lu_f64_2048"):
        n = 2048
        Q = torch.from_numpy(synth.dct2_matrix(n)).cuda()
        LUb = torch.empty_like(Q)
        ipiv = torch.empty(n, dtype=torch.int32, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")

        def restore_and_flush():  # untimed: the factorisation is in place
            LUb.copy_(Q)
            flush()
        ms = timed_steps(torch, lambda: fb.fb_lu(LUb, ipiv, info, stream), steps, args.warmup, restore_and_flush,
                         stream)
        t = float(np.mean(ms))
        flops = 2.0 / 3.0 * n ** 3
        res["lu_f64_2048"] = {"value": flops / (t * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": t,
                              "config": {"workload": "lu_2048_fp64_orthogonal_dct2", "survey_next": "N2",
                                         "flops": "2/3 n^3"},
                              "note": "look-ahead: one-CTA 8-column panels (pivot search by redux.sync) overlap "
                                      "the swap/TRSM + streaming rank-8 update of the previous step on a second "
                                      "stream; latency-bound by the 2048 sequential pivot steps"}
        del Q, LUb
    # configs[0]: 256^2 forward + inverse
    if want("fft2d_256_fwd_inv"):
        m = 256
        x = torch.from_numpy(synth.complex_field(m, m)).cuda()
        y = torch.empty_like(x)
        z = torch.empty_like(x)

        wsb = fb.lib().fb_fft2d_workspace_bytes(m, m)
        ws2 = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda") if wsb else None

        def fi():
            fb.fb_fft2d(x, y, ws2, stream)
            fb.fb_ifft2d(y, z, ws2, stream)
        ms = timed_steps(torch, fi, steps, args.warmup, flush, stream)
        t = float(np.mean(ms))
        res["fft2d_256_fwd_inv"] = {"value": 2 * fft_flops(m, m) / (t * 1e-3) / 1e9, "unit": "GFLOP/s",
                                    "ms_per_step": t, "config": {"workload": "fft2d_256x256_fwd+inv",
                                                                 "configs_index": 0}}
    # single-GPU 16384^2 forward: the N=1 point of the configs[3] scaling series
    if want("fft2d_16384"):
        m = 16384
        x = torch.from_numpy(synth.complex_field(m, m)).cuda()
        y = torch.empty_like(x)
        ws = torch.empty(fb.lib().fb_fft2d_workspace_bytes(m, m), dtype=torch.uint8, device="cuda")
        ms = timed_steps(torch, lambda: fb.fb_fft2d(x, y, ws, stream), steps, args.warmup, flush, stream)
        t = float(np.mean(ms))
        passes = 2  # the algorithmic traffic is 2 passes x (R + W) = 8 GiB at P = 1
        ach = passes * 2 * 8 * m * m / (t * 1e-3) / 1e9
        res["fft2d_16384"] = {"value": fft_flops(m, m) / (t * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": t,
                              "config": {"workload": "fft2d_16384x16384_fwd_1gpu", "configs_index": 3},
                              "roofline": {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                           "frac": ach / pk["hbm_gbs"],
                                           "traffic_row_pass": ncu_traffic("fft2d_16384"),
                                           "note": "algorithmic 2 passes x (R+W) of the 2 GiB array = 8 GiB "
                                                   "(SURVEY 8(d)); the implementation moves 3 passes (four-step "
                                                   "16384-long columns)"}}
        del x, y, ws
    if want("gemm_bf16_8192"):  # N4: BF16 operands, FP32 accumulation (roofline: measured BF16 peak)
        n = 8192
        g = torch.Generator(device="cuda").manual_seed(200409885)
        A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        Bt = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
        C = torch.empty(n, n, device="cuda")
        ms = timed_steps(torch, lambda: fb.matmul_bf16(A, Bt, b_transposed=True, out=C, stream=stream), steps,
                         args.warmup, flush, stream)
        t = float(np.mean(ms))
        tf = 2.0 * n ** 3 / (t * 1e-3) / 1e12
        res["gemm_bf16_8192"] = {"value": tf, "unit": "TFLOP/s", "ms_per_step": t,
                                 "config": {"workload": "gemm_8192^3_bf16_fp32acc", "survey_next": "N4",
                                            "b_layout": "K-major (B^T given)"},
                                 "roofline": {"bound": "tensor", "achieved": tf, "peak": pk["bf16_tflops"],
                                              "unit": "TFLOP/s", "frac": tf / pk["bf16_tflops"],
                                              "traffic": ncu_traffic("gemm_bf16_8192"),
                                              "peak_source": pk["source"] + " (BF16 burst)"}}
        del A, Bt, C
    if want("gemm_f32_32768"):  # configs[4] at 1 GPU: the scaling baseline of the row-block GEMM
        res["gemm_f32_32768"] = rowblock_gemm(args, torch, fb, np, stream, flush, pk, None, 0, 1, None)
    return res


def rowblock_gemm(args, torch, fb, np, stream, flush, pk, dist, rank, world, comm):
    """configs[4]: C = A B, 32768^3 FP32 (3xTF32), A and C row-sharded over `world` ranks, B broadcast
    from rank 0 inside the timed region (fb_matmul_rowblock; plain fb_matmul at world size 1)."""
    n = 32768
    rows = n // world
    g = torch.Generator(device="cuda").manual_seed(200409883 + rank)
    A = (torch.rand(rows, n, device="cuda", generator=g) * 2 - 1)
    B = (torch.rand(n, n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(200409884)) * 2 - 1)
    C = torch.empty(rows, n, device="cuda")
    if comm is None:
        ws = torch.empty(fb.matmul_workspace_bytes(fb.FB_F32, rows, n, n), dtype=torch.uint8, device="cuda")
        fn = lambda: fb.fb_matmul(A, B, C, ws, stream)  # noqa: E731
    else:
        ws = torch.empty(fb.lib().fb_matmul_rowblock_workspace_bytes(world, fb.FB_F32, n, n, n), dtype=torch.uint8,
                         device="cuda")
        fn = lambda: comm.fb_matmul_rowblock(A, B, C, root=0, ws=ws, stream=stream)  # noqa: E731
    ms = timed_steps(torch, fn, 3, min(args.warmup, 3), flush, stream, dist)
    t = max_over_ranks(torch, dist, float(np.mean(ms)))
    del A, B, C, ws
    flops = 2.0 * n * n * n
    tf32_peak = tc_peaks()["tf32_sustained"]
    return {"value": flops / (t * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": t,
            "config": {"workload": "gemm_32768^3_fp32_3xtf32_rowblock", "configs_index": 4,
                       "parallelism": f"rowblock{world}", "data": "uniform [-1, 1) (torch, seeded, on device)",
                       "b_broadcast": ("N-column panels (FB_ROWBLOCK_PANEL) broadcast inside the timed region, "
                                       "each panel's GEMM overlapping the next panel's broadcast")
                       if comm is not None else "none"},
            "roofline": {"bound": "tensor", "achieved": 3 * flops / world / (t * 1e-3) / 1e12, "peak": tf32_peak,
                         "unit": "TFLOP/s", "frac": 3 * flops / world / (t * 1e-3) / 1e12 / tf32_peak,
                         "note": "per GPU, counting the 3 TF32 MMAs (6MNK/P), split pre-pass and broadcast "
                                 "inside the time; peak = measured sustained TF32 (profiles/r2_peaks.json)"}}


def run_slab(args, torch, fb, synth, np, stream, flush, pk, dist, rank, world, local):
    """configs[3]: 16384^2 FFT slab-sharded over `world` ranks (fused NVLink transpose, or one NCCL
    all-to-all when the fused path is unavailable)."""
    n = 16384
    rows = n // world
    x = torch.from_numpy(synth.complex_field(n, n, row0=rank * rows, rows=rows)).cuda()
    y = torch.empty(n, n // world, dtype=torch.complex64, device="cuda")
    comm = fb.Comm(rank, world, local)
    ws = torch.empty(fb.lib().fb_fft2d_slab_workspace_bytes(world, n, n), dtype=torch.uint8, device="cuda")
    L0 = fb.launch_count()
    with ClockSampler(local) as clk:
        ms = timed_steps(torch, lambda: comm.fb_fft2d_slab(x, y, n, n, ws, stream), args.steps, args.warmup, flush,
                         stream, dist)
    launches = (fb.launch_count() - L0) // (args.steps + args.warmup)
    t = max_over_ranks(torch, dist, float(np.mean(ms)))
    # e2e: each rank's slab from pinned host memory -> fb_fft2d_slab -> column slab back to the host
    xh = torch.empty(rows, n, dtype=torch.complex64, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.empty(n, n // world, dtype=torch.complex64, pin_memory=True)

    def e2e_step():
        x.copy_(xh, non_blocking=True)
        comm.fb_fft2d_slab(x, y, n, n, ws, stream)
        yh.copy_(y, non_blocking=True)

    me = timed_steps(torch, e2e_step, max(2, args.steps // 2), args.warmup, flush, stream, dist)
    te = max_over_ranks(torch, dist, float(np.mean(me)))
    fused = comm.fused
    del xh, yh, x, y, ws
    gemm = rowblock_gemm(args, torch, fb, np, stream, flush, pk, dist, rank, world, comm)
    comm.destroy()
    val = fft_flops(n, n) / (t * 1e-3) / 1e9
    hbm = 2 * 2 * 8 * n * n / world  # 2 local passes x (R+W) per GPU (8/4/2/1 GiB)
    ach = hbm / (t * 1e-3) / 1e9
    return {"value": val, "unit": "GFLOP/s", "ms_per_step": t, "scaling": "strong",
            "config": {"workload": "fft2d_16384x16384_slab", "n0": n, "n1": n, "configs_index": 3,
                       "parallelism": f"slab{world}",
                       "l2": "inputs (2 GiB total) larger than L2; L2 also flushed before every step"},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": ach / pk["hbm_gbs"],
                         "note": "per-GPU local HBM passes only (the transpose's NVLink traffic is not counted)"},
            "transpose": "fused NVLink (NCCL symmetric windows + LSA barriers)" if fused else "ncclAlltoAll",
            "e2e": {"value": fft_flops(n, n) / (te * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": te,
                    "h2d_bytes_per_step": rows * n * 8, "d2h_bytes_per_step": n * (n // world) * 8,
                    "api": "pinned torch copies + fb_fft2d_slab, per rank"},
            "gpu_launches": launches * args.steps, "clocks": clk.summary(),
            "blocks": {"gemm_f32_32768_rowblock": gemm}}


if __name__ == "__main__":
    sys.exit(main())
