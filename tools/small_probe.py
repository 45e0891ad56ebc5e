"""Per-iteration timing of the latency-bound configs (C1, C2, C3) through the
public API; run under `ncu --metrics gpu__time_duration.sum` for the launch
list.  Usage: python tools/small_probe.py [C1|C2|C3 ...] [--iters N]"""
import argparse
import sys
import time

sys.path.insert(0, "/root/repo")
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402
from paper_1409_7474_b200.bands import BandEvolutionRun  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3"])
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

for cfg in a.configs:
    if cfg == "C3":
        sc = scenes.config3(4096, a.iters or 1000)
        mk = lambda: BandEvolutionRun(sc.image, sc.extra["signs"],  # noqa: E731
                                      L.default_params(L.ModelKind.REGION, **sc.params))
    else:
        # C1, C2, or X<size>: a C5-density crop of that side, 200 iterations
        sc = (scenes.config1() if cfg == "C1" else scenes.config2() if cfg == "C2"
              else scenes.config5_crop(int(cfg[1:]), 200))
        kind = L.ModelKind.from_name(sc.model)
        mk = lambda: L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),  # noqa: E731
                                    L.default_params(kind, **sc.params))
    n = a.iters or sc.iters
    for rep in range(a.reps):
        r = mk()
        r.set_native_option("skip_uniform", 0)
        t0 = time.perf_counter()
        r.advance(n)
        dt = time.perf_counter() - t0
        print(f"{cfg} rep {rep}: {n} its, {dt / n * 1e6:.1f} us/it (wall, incl. sync)", flush=True)
