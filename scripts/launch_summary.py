"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per kernel, the number
of launches, total / mean duration and share of all kernel time.  Usage: launch_summary.py CSV."""
import csv
import sys
from collections import defaultdict

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in csv.DictReader(rows):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}[r["Metric Unit"]]
    name = r["Kernel Name"].split("(")[0]
    tot[name] += v * scale
    cnt[name] += 1
allt = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean ms':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:10.3f} {tot[k] / cnt[k]:10.4f} {tot[k] / allt * 100:6.1f}%")
print(f"{'all':60s} {sum(cnt.values()):8d} {allt:10.3f}")
