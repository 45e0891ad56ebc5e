import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from paper_1409_7474_b200.batch import TileBatch, _tile_run
T, iters = 32, 300
sc = [scenes.config4_tile(k % 16, 1024, iters) for k in range(T)]
runs = [_tile_run(s.image, L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign),
                  L.default_params(L.ModelKind.from_name(s.model), **s.params)) for s in sc]
for r in runs: r.set_native_option("skip_uniform", 0)
tb = TileBatch(runs)
for chunk in (10, 40, 250):
    t0 = time.perf_counter(); tb.advance(chunk); dt = time.perf_counter() - t0
    st = [r.spec_stats() for r in runs]
    print(f"chunk {chunk}: {dt*1e3:.1f} ms, redos per tile {[s['redos'] for s in st[:8]]}, fixes {[s['fixes'] for s in st[:8]]}, it {[r.state.iteration for r in runs[:8]]}, conv {[r.state.converged for r in runs[:8]]}", flush=True)
