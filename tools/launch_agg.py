"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows:
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        a = agg.setdefault(r[ki].split("(")[0].replace("void ", "")[:48], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(t for _, t in agg.values())
    print(f"== {path}  total {tot:.1f} us")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} {n:5d} {t / n:9.2f} us  {100 * t / tot:5.1f}%")
