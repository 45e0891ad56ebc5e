"""C3 timing probe (4 bands)."""
import sys
import time
sys.path.insert(0, "/root/repo")
import numpy as np  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402
from paper_1409_7474_b200.bands import BandEvolutionRun  # noqa: E402
size, iters = int(sys.argv[1]), int(sys.argv[2])
sc = scenes.config3(size, iters)
r = BandEvolutionRun(sc.image, sc.extra["signs"], L.default_params(L.ModelKind.REGION, **sc.params))
r.set_native_option("skip_uniform", 0)
t0 = time.perf_counter()
r.advance(iters)
print(size, iters, (time.perf_counter() - t0) / iters * 1e3, "ms/it")
