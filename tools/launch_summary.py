"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total time and share per kernel.  python tools/launch_summary.py <csv>"""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        if x.get("Metric Name") == "gpu__time_duration.sum":
            us = float(x["Metric Value"].replace(",", "")) * SCALE[x["Metric Unit"]]
            k = x["Kernel Name"].split("(")[0].strip()[:80]
            agg[k][0] += 1
            agg[k][1] += us
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total us':>12} {'share':>6}  kernel")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {us:12.1f} {100 * us / tot:5.1f}%  {k}")
