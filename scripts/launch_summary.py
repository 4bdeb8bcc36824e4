"""Per-launch table of an ncu --csv launch list (gpu__time_duration, DRAM bytes; tensor pipe when present): the last
`--last` launches, and their total time."""
import argparse
import collections
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--last", type=int, default=40)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    per.setdefault((int(r[ii]), r[ki][:64]), {})[r[mi]] = r[vi].replace(",", "")
tot = 0.0
for (i, k), m in list(per.items())[-a.last:]:
    t = float(m["gpu__time_duration.sum"]) / 1e3
    tot += t
    rd = float(m.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(m.get("dram__bytes_write.sum", 0)) / 1e6
    tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "")
    print(f"{i:4d} {k:64s} {t:9.1f} us  R {rd:9.1f} MB  W {wr:8.1f} MB {tp}")
print(f"total {tot:.1f} us")
