"""Near-tie fp64 re-evaluations per iteration for the BASELINE configs."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402

for cfg in sys.argv[1:] or ["C1", "C2"]:
    sc = scenes.config1() if cfg == "C1" else scenes.config2() if cfg == "C2" else \
        scenes.config5_crop(int(cfg[1:]), 200)
    kind = L.ModelKind.from_name(sc.model)
    r = L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),
                       L.default_params(kind, **sc.params))
    r.advance(sc.iters)
    n = r.fallback_count()
    print(cfg, sc.image.shape, "iterations", sc.iters, "exact fallbacks", n,
          "per iteration", n / sc.iters)
