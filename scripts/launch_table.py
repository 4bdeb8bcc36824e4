"""Dev: per-iteration kernel times from an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
r = list(csv.reader(lines))
h = r[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = collections.OrderedDict(), collections.Counter()
for row in r[1:]:
    if len(row) <= iv:
        continue
    name = row[ik].split("(")[0].replace("void ", "").strip()
    tot[name] = tot.get(name, 0.0) + float(row[iv].replace(",", ""))
    cnt[name] += 1
iters = cnt["lfm::metric_sum_kernel"] or cnt["lfm::metric_final_kernel"]
rows = [(tot[n] / cnt[n] / 1e6, n, cnt[n]) for n in tot if cnt[n] in (iters, iters + 1)]
step = sum(x[0] for x in rows)
for ms, n, c in sorted(rows, reverse=True):
    print(f"{ms:8.4f} ms  {ms / step * 100:5.1f}%  {n} x{c}")
print(f"sum {step:.3f} ms over {iters} iterations")
