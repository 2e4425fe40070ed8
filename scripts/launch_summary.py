"""Aggregate an ncu launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
rd = csv.DictReader(lines)
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    scale = {"ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(unit, 1e-9)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print(f"total device time {T:.4f} s over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.4f} s  {100 * v / T:5.1f}%  {cnt[k]:7d} launches  {k}")
