"""Wall-clock breakdown of the drop-in run() on the C5 scene: run creation
(pageable image upload), advance, mask read-back, teardown."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LSE_SKIP_UNIFORM"] = "0"
import numpy as np  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402

size = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
sc = scenes.config5(size=size, n_rects=20000, iters=500)
img = np.array(sc.image, dtype=np.float32)
seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
prm = L.default_params(L.ModelKind.REGION, **sc.params)
for rep in range(3):
    t0 = time.perf_counter()
    r = L.EvolutionRun(img, seeds, prm)
    t1 = time.perf_counter()
    r.advance(500)
    t2 = time.perf_counter()
    m = r.mask()
    t3 = time.perf_counter()
    del r
    t4 = time.perf_counter()
    print(f"rep {rep}: create {t1 - t0:.3f} s, advance {t2 - t1:.3f} s, mask {t3 - t2:.3f} s, "
          f"destroy {t4 - t3:.3f} s, total {t4 - t0:.3f} s ({m.dtype}, {m.sum()} px inside)", flush=True)
