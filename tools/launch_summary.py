#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list CSV (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
n = 0
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    unit = d.get("Metric Unit", "ns")
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    nm = d["Kernel Name"].split("(")[0].strip()
    a = agg[nm]
    a[0] += 1
    a[1] += v
    n += 1
tot = sum(a[1] for a in agg.values())
print(f"# {n} launches, kernel time {tot:.1f} ms (serialised, cold-cache)")
print(f"{'kernel':70s} {'launches':>9s} {'total ms':>10s} {'share':>7s} {'mean us':>9s}")
for nm, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{nm[:70]:70s} {c:9d} {t:10.2f} {100 * t / tot:6.2f}% {1e3 * t / c:9.2f}")
