"""Per-kernel share of the device time in an ncu --metrics gpu__time_duration.sum launch list (CSV).

    python tools/launch_shares.py launches.csv            # every launch in the list
    python tools/launch_shares.py launches.csv --step 2   # only the launches of the 2nd training step

The loss reduction (`sum_f64_kernel`) runs once per tawpipe step, after the head, so the launches after the
(k-1)-th and up to the k-th `sum_f64_kernel` are one step's worth of work (the backward of step k-1 and the forward
of step k, k >= 2); window 1 holds the initialisation and the first forward only."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
step = int(sys.argv[sys.argv.index("--step") + 1]) if "--step" in sys.argv else 0
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
launches = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:60]
    launches.append((name, v))
if step:
    ends = [i for i, (n, _) in enumerate(launches) if "sum_f64_kernel" in n]
    if len(ends) < step:
        sys.exit(f"only {len(ends)} complete step(s) in the list")
    lo = ends[step - 2] + 1 if step > 1 else 0
    launches = launches[lo:ends[step - 1] + 1]
tot, cnt = collections.defaultdict(float), collections.Counter()
for name, v in launches:
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
what = f"one-step window {step}" if step else "all launches"
print(f"{what}: total {T:.1f} ms over {sum(cnt.values())} launches (ncu: serialised, cold cache)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.2f} ms {100 * v / T:6.2f}% {cnt[k]:6d}  {k}")
