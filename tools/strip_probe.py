"""Per-strip kernel times of a G-strip decomposition of C5, emulated on one GPU
(LocalComm): what each rank of a G-GPU run would spend per iteration."""
import ctypes as C
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
from paper_1409_7474_b200 import _native as N, scenes, default_params, ModelKind, SeedSpec  # noqa: E402
from paper_1409_7474_b200.strips import DeviceStrip, LocalComm, StripDriver, plan_strips  # noqa: E402

size, world, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n_rects = max(1, int(round(20000 * (size / 32768.0) ** 2)))
wins = plan_strips(size, size, world)
strips = []
for w in wins:
    sc = scenes.config5(size, n_rects, iters, rows=(w.y_lo, w.y_hi))
    prm = default_params(ModelKind.REGION, **sc.params)
    strips.append(DeviceStrip(sc.image, w, SeedSpec(polygons=sc.polygons,
                                                    inside_sign=sc.inside_sign), prm))
    del sc
for s in strips:
    N.check(N.lib.lse_run_set_option(s.h, b"skip_uniform", 0))
# serialize the strips' kernels (each strip alone on the GPU, as on its own rank)
for s in strips:
    for name in ("update", "partition", "finalize"):
        f = getattr(s, name)

        def wrapped(*a, _f=f, _s=s, **k):
            r = _f(*a, **k)
            _s.synchronize()
            return r
        setattr(s, name, wrapped)
drv = StripDriver(strips, LocalComm(strips))
drv.setup()
drv.advance(3)
for s in strips:
    N.check(N.lib.lse_run_set_profiling(s.h, 1))
t0 = time.perf_counter()
drv.advance(iters)
dt = time.perf_counter() - t0
for k, s in enumerate(strips):
    u, p, nu, np_ = C.c_double(), C.c_double(), C.c_longlong(), C.c_longlong()
    N.check(N.lib.lse_run_kernel_times(s.h, C.byref(u), C.byref(nu), C.byref(p), C.byref(np_)))
    print(f"strip {k}: rows {wins[k].own_rows} update {u.value / max(1, nu.value):.4f} ms "
          f"partition {p.value / max(1, np_.value):.4f} ms")
print(f"wall {dt / iters * 1e3:.3f} ms/it (LocalComm syncs, not representative)")
