"""Sum an ncu --csv metrics log per kernel name over the last `tail` launches.
usage: python tools/ncu_csv_sum.py log.csv [tail]"""
import collections
import csv
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3}
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h, rows = rows[0], rows[1:]
iid, ik, im, iv, iu = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.OrderedDict()
for r in rows:
    per.setdefault(r[iid], {"k": r[ik][:70]})[r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1)
ids = list(per)
tail = int(sys.argv[2]) if len(sys.argv) > 2 else len(ids)
tot = collections.OrderedDict()
for i in ids[-tail:]:
    d = per[i]
    t = tot.setdefault(d["k"], collections.defaultdict(float))
    t["n"] += 1
    for m, v in d.items():
        if m != "k":
            t[m] += v
print(f"{len(ids)} launches, last {tail}:")
for k, t in tot.items():
    print(f"  {k:70s} n={int(t['n'])} t={t['gpu__time_duration.sum']:.1f}us "
          f"rd={t['dram__bytes_read.sum'] / 1e6:.0f}MB wr={t['dram__bytes_write.sum'] / 1e6:.0f}MB")
