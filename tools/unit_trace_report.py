"""Summarize an LSE_UNIT_TRACE_FILE: per launch, kernel span, the slowest
units (border vs interior), and the busy-warp profile."""
import sys

import numpy as np

for line in open(sys.argv[1]):
    line, _, ex = line.partition("|")
    e = ex.split()
    f = line.split()
    name, n, nb, grid = f[0], int(f[1]), int(f[2]), int(f[3])
    allv = np.array(f[4:], dtype=np.int64).reshape(n + grid, 2)
    a, cta = allv[:n], allv[n:]
    cok = cta[:, 0] >= 0
    print(f"  CTA entry: first {cta[cok,0].min()/1e3:.1f} last {cta[cok,0].max()/1e3:.1f} us; "
          f"entry->first grab mean {(cta[cok,1]-cta[cok,0]).mean()/1e3:.1f} max "
          f"{(cta[cok,1]-cta[cok,0]).max()/1e3:.1f} us")
    ok = (a[:, 0] >= 0) & (a[:, 1] >= 0)
    dur = (a[:, 1] - a[:, 0])
    span = a[ok, 1].max()
    b, i = dur[:nb][ok[:nb]], dur[nb:][ok[nb:]]
    print(f"{name}: units {n} (border {nb}) span {span/1e3:.1f} us | "
          f"border mean {b.mean()/1e3 if b.size else 0:.1f} max {b.max()/1e3 if b.size else 0:.1f} us | "
          f"interior mean {i.mean()/1e3 if i.size else 0:.1f} p99 {np.percentile(i, 99)/1e3 if i.size else 0:.1f} "
          f"max {i.max()/1e3 if i.size else 0:.1f} us | "
          f"last start {a[ok,0].max()/1e3:.1f} us")
    if e:
        print(f"   warps exit by {int(e[2])/1e3:.1f} us; stamps before {int(e[4])/1e3:.1f} "
              f"after {int(e[5])/1e3:.1f} us (kernel wall ~{(int(e[5]) - int(e[4]))/1e3:.1f} us)")
    worst = np.argsort(-dur)[:5]
    print("   slowest:", [(int(u), "B" if u < nb else "I", round(dur[u] / 1e3, 1), round(a[u, 0] / 1e3, 1)) for u in worst])
