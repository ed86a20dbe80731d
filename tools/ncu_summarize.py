"""Summarise ncu reports into small committed text/JSON files under profiles/.

usage: python tools/ncu_summarize.py REPORT.ncu-rep OUT_PREFIX [WORKLOAD KERNEL_SUBSTR [KEY]]
Writes OUT_PREFIX.txt (per-kernel key metrics) and merges dram bytes per launch into
profiles/ncu_traffic.json (keyed by workload tag inferred from the kernel name).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_us"),
    ("dram__bytes_read.sum", "dram_read_MB"),
    ("dram__bytes_write.sum", "dram_write_MB"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc_inst_pct"),
    # tcgen05 (UMMA) tensor-core activity; the *_realtime "tensor_pipe" counter above does not
    # track tcgen05.mma on sm_100
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "umma_active_pct"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_inst_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
]


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0, "GB": 1e3}
    lines = [f"# ncu --set full summary of {os.path.basename(rep)} (units: us, MB, %)"]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        lines.append(name[:110])
        vals = {}
        for k, label in KEYS:
            if k in hdr and r[hdr.index(k)] not in ("", "n/a"):
                v = r[hdr.index(k)]
                u = units[hdr.index(k)]
                if label.endswith("_MB") and u in scale:  # normalise to MB whatever unit ncu chose
                    v = "%.3f" % (float(v.replace(",", "")) * scale[u])
                elif k == "gpu__time_duration.sum" and u in ("ns", "us", "ms", "msecond", "usecond", "nsecond"):
                    f = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[u]
                    v = "%.3f" % (float(v.replace(",", "")) * f)
                vals[label] = v
        lines.append("    " + "  ".join(f"{k}={v}" for k, v in vals.items()))
        try:
            rd = float(vals.get("dram_read_MB", "0").replace(",", ""))
            wr = float(vals.get("dram_write_MB", "0").replace(",", ""))
            short = name.split("(")[0].replace("void ", "").strip()
            traffic.setdefault(short, []).append((rd + wr) * 1e6)
        except ValueError:
            pass
    open(prefix + ".txt", "w").write("\n".join(lines) + "\n")
    tp = os.path.join(os.path.dirname(prefix) or ".", "ncu_traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    for k, v in traffic.items():
        cur.setdefault("per_kernel_bytes", {})[k] = sum(v) / len(v)
    if len(sys.argv) > 4:  # workload tag + kernel-name substring: mean bytes per launch of those kernels
        tag, sub = sys.argv[3], sys.argv[4]
        vs = [x for k, v in traffic.items() if sub in k for x in v]
        if vs:
            cur.setdefault(tag, {})[sys.argv[5] if len(sys.argv) > 5 else sub] = sum(vs) / len(vs)
    json.dump(cur, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
