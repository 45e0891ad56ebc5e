"""ncu --csv launch list with gpu__time_duration.sum (+ optionally
dram__bytes_read/write.sum) -> per-kernel table: launches, median / min / max
duration, share of the total time, median DRAM MB read / written."""
import collections
import csv
import statistics
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
SC = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
      "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
agg = collections.OrderedDict()
for r in rows:
    name = r[ki].split("(")[0].replace("void ", "")[:44]
    v = float(r[vi].replace(",", "")) * SC.get(r[ui], 1.0)
    agg.setdefault(name, collections.defaultdict(list))[r[mi]].append(v)
tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
print(f"{'kernel':44s} {'n':>5s} {'median us':>10s} {'min':>9s} {'max':>9s} {'share':>6s} {'DRAM rd MB':>10s} {'wr MB':>8s}")
for k, m in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
    t = m["gpu__time_duration.sum"]
    rd = m.get("dram__bytes_read.sum")
    wr = m.get("dram__bytes_write.sum")
    print(f"{k:44s} {len(t):5d} {statistics.median(t):10.2f} {min(t):9.2f} {max(t):9.2f} "
          f"{100 * sum(t) / tot:5.1f}% "
          f"{statistics.median(rd) if rd else float('nan'):10.1f} {statistics.median(wr) if wr else float('nan'):8.1f}")
