"""C4 timing probe: T tiles of 1024^2 8-bit RGB, batched, `iters` iterations."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402
from paper_1409_7474_b200.batch import TileBatch, _tile_run  # noqa: E402

T, size, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
t0 = time.perf_counter()
sc = [scenes.config4_tile(k % 16, size, iters) for k in range(T)]   # 16 distinct tiles, reused
t_gen = time.perf_counter() - t0
t0 = time.perf_counter()
runs = [_tile_run(s.image, L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign),
                  L.default_params(L.ModelKind.from_name(s.model), **s.params)) for s in sc]
t_create = time.perf_counter() - t0
for r in runs:
    r.set_native_option("skip_uniform", 0)
t0 = time.perf_counter()
tb = TileBatch(runs)
t_batch = time.perf_counter() - t0
t0 = time.perf_counter()
tb.advance(iters)
t_adv = time.perf_counter() - t0
px_its = T * size * size * iters
print(f"T={T} size={size} iters={iters}: gen {t_gen:.2f}s create {t_create:.2f}s "
      f"batch {t_batch:.2f}s advance {t_adv*1e3:.1f} ms -> {px_its / t_adv / 1e9:.1f} Gpix-it/s")
