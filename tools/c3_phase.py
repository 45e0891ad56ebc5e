"""C3 per-phase timing: ms per iteration in chunks over the 1000-iteration
job (the checkerboard partition settles within ~40 iterations), with and
without the peak-pass reuse."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402
from paper_1409_7474_b200.bands import BandEvolutionRun  # noqa: E402

size, iters, chunk = (int(a) for a in (sys.argv[1:4] + ["4096", "1000", "50"][len(sys.argv[1:4]):]))
sc = scenes.config3(size, iters)
prm = L.default_params(L.ModelKind.REGION, **sc.params)
for reuse in ("1", "0"):
    os.environ["LSE_BAND_REUSE"] = reuse
    r = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r.set_native_option("skip_uniform", 0)
    r.advance(2)
    r.state.iteration
    out = []
    t_all = time.perf_counter()
    done = 2
    while done < iters:
        n = min(chunk, iters - done)
        t0 = time.perf_counter()
        r.advance(n)
        r.state.iteration
        out.append(round((time.perf_counter() - t0) / n * 1e3, 4))
        done += n
    tot = time.perf_counter() - t_all
    print(f"reuse={reuse} {size}^2 x {iters}: {tot / (iters - 2) * 1e3:.4f} ms/it "
          f"({size * size * (iters - 2) / tot / 1e9:.1f} Gpix-it/s) {r.band_stats()}")
    print("  per chunk ms/it:", out)
