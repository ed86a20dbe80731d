"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel.

usage: python tools/launch_summary.py LAUNCHES.csv OUT_PREFIX "command that was profiled"
Writes OUT_PREFIX_summary.txt (kernel | launches | mean_ns | total_ns, plus each libfb kernel's
share of the libfb total) and OUT_PREFIX.csv (the launch rows of libfb's own kernels only)."""
import collections
import csv
import sys

src, prefix, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
agg = collections.OrderedDict()
ours = []
OURS = ("fb::", "lu::", "tf32::", "f64::", "pair::", "fft_", "gemm_", "lu_", "split_", "lsa_", "bs_", "rfft_", "scale_kernel")
for r in rows[start + 1:]:
    if len(r) <= max(ki, mi, vi) or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki]
    short = name.split("(")[0].replace("void ", "").strip()
    t = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg.setdefault(short, []).append(t)
    if any(o in name for o in OURS):
        ours.append((short, t))
mine = {k: v for k, v in agg.items() if any(o in k for o in OURS)}
tot_mine = sum(sum(v) for v in mine.values()) or 1.0
lines = ["# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
         "# command: " + cmd, "# kernel | launches | mean_ns | total_ns | share of libfb kernel time"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = "%.1f%%" % (100 * sum(v) / tot_mine) if k in mine else "-"
    lines.append(f"{k[:90]} | {len(v)} | {sum(v) / len(v):.0f} | {sum(v):.0f} | {share}")
open(prefix + "_summary.txt", "w").write("\n".join(lines) + "\n")
with open(prefix + ".csv", "w") as f:
    f.write("kernel,duration_ns\n")
    for k, t in ours:
        f.write(f'"{k}",{t:.0f}\n')
print("\n".join(lines[:40]))
