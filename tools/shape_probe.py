"""Per-iteration kernel times of a single run on a C5-density scene of a given
shape (rows x 32768 columns by default): fused pass vs two-pass iteration.

    python tools/shape_probe.py ROWS [COLS] [ITERS]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1409_7474_b200 import _native as N, scenes, default_params, ModelKind, SeedSpec  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402

rows = int(sys.argv[1])
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 60
sc = scenes.config5(cols, 20000, iters, rows=(0, rows))
prm = default_params(ModelKind.REGION, **sc.params)
for fused in ("1", "0"):
    os.environ["LSE_FUSED"] = fused
    r = L.EvolutionRun(sc.image, SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign), prm)
    r.set_native_option("skip_uniform", 0)
    r.advance(10)
    N.check(N.lib.lse_run_set_profiling(r._dev.h, 1))
    r.advance(iters - 10)
    u, p, nu, np_ = C.c_double(), C.c_double(), C.c_longlong(), C.c_longlong()
    N.check(N.lib.lse_run_kernel_times(r._dev.h, C.byref(u), C.byref(nu), C.byref(p), C.byref(np_)))
    print(f"{rows}x{cols} fused={fused}: update {1e3 * u.value / max(1, nu.value):8.1f} us, "
          f"partition/finalize {1e3 * p.value / max(1, np_.value):7.1f} us per iteration "
          f"({nu.value} / {np_.value} launches)", flush=True)
