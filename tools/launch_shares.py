"""Per-kernel share of the device time in an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:60]
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.1f} ms over {sum(cnt.values())} launches (ncu: serialised, cold cache)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.2f} ms {100 * v / T:6.2f}% {cnt[k]:6d}  {k}")
