"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r["Metric Unit"]] * v
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:44]:44s} {v[0]:8d} {v[1]:10.1f} {v[1] / v[0]:8.2f} {100 * v[1] / tot:5.1f}%")
print(f"total {tot:.1f} us over {len(rows)} launches")
