"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
count, total time and share.  usage: python tools/launch_summary.py launches.csv"""
import csv
import io
import sys
from collections import defaultdict

txt = open(sys.argv[1]).read()
start = txt.find('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = defaultdict(lambda: [0, 0.0])
total = 0.0
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
    name = r["Kernel Name"].split("(")[0][:90]
    agg[name][0] += 1
    agg[name][1] += v
    total += v
print(f"{'kernel':90s} {'n':>6s} {'us':>10s} {'share':>6s}")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:90s} {n:6d} {us:10.1f} {100 * us / total:5.1f}%")
print(f"total {total:.1f} us over {sum(n for n, _ in agg.values())} launches")
