"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time per kernel name."""
import collections
import csv
import sys

path = sys.argv[1]
solves = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'ms/solve':>10} {'share':>6} {'launches':>8}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v / solves:10.3f} {100 * v / T:5.1f}% {cnt[k] / solves:8.0f}  {k}")
print(f"{T / solves:10.3f} total (ncu: serialised, cold-cache per launch)")
