#!/usr/bin/env python
"""Guard certification of the fp32 fast path on a BASELINE workload.

Loads the validation build (liblse_b200_check.so, `make check`), in which the
fused update / partition kernels also evaluate every pixel's decision value
in the reference's fp64 operation order (exact_u_fast / exact_phi_fast) and
record, per thread, max |u32 - u64| / eps_u, max |phi32 - phi64| / eps_phi,
the smallest |u64| / |phi64| seen (how close the closest decision came to a
tie) and the number of fp32 decisions outside the guard band that disagree
with fp64 (must be 0).  Every decision of the product build is then provably
the reference's fp64 decision when both ratios stay below 1.

  python tools/certify.py --config C5 [--size 32768] [--iters 500] [--every 1]

prints one JSON line (and writes it to --out when given).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
import warnings

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(REPO, "paper_1409_7474_b200", "_lib", "liblse_b200_check.so")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--every", type=int, default=1, help="check every k-th iteration")
    ap.add_argument("--tiles", type=int, default=16, help="C4: tiles in the batch")
    ap.add_argument("--skip-uniform", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.environ["LSE_LIB_PATH"] = CHECK_LIB
    os.environ["LSE_CHECK_EVERY"] = str(a.every)
    sys.path.insert(0, REPO)
    import numpy as np
    import paper_1409_7474_b200 as L
    from paper_1409_7474_b200 import _native as N, scenes
    if not N.lib.lse_check_enabled():
        raise SystemExit("not the certification build")

    def prm(model, **kw):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return L.default_params(L.ModelKind.from_name(model), **kw)

    t0 = time.perf_counter()
    cfg = a.config
    if cfg == "C5":
        size = a.size or 32768
        iters = a.iters or 500
        sc = scenes.config5(size=size, n_rects=max(1, int(round(20000 * (size / 32768) ** 2))),
                            iters=iters)
        runs = [L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons,
                                                    inside_sign=sc.inside_sign),
                               prm("region", **sc.params))]
        npx = size * size
        desc = f"C5 {size}^2 region, sigma 1.5 (9x9), dt 15, {iters} its"
    elif cfg == "C3":
        from paper_1409_7474_b200.bands import BandEvolutionRun
        size = a.size or 4096
        iters = a.iters or 1000
        sc = scenes.config3(size, iters)
        runs = [BandEvolutionRun(sc.image, sc.extra["signs"], prm("region", **sc.params))]
        npx = size * size
        desc = f"C3 {size}^2 x 4 bands, {iters} its"
    elif cfg == "C4":
        from paper_1409_7474_b200.batch import _tile_run
        size = a.size or 1024
        iters = a.iters or 300
        scs = [scenes.config4_tile(k, size, iters) for k in range(a.tiles)]
        runs = [_tile_run(s.image, L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign),
                          prm(s.model, **s.params)) for s in scs]
        npx = size * size * a.tiles
        desc = f"C4 tiles 0..{a.tiles - 1}, {size}^2 RGB, region/edge, {iters} its, one batch"
    else:
        sc = scenes.config1() if cfg == "C1" else scenes.config2()
        iters = a.iters or sc.iters
        runs = [L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons,
                                                    inside_sign=sc.inside_sign),
                               prm(sc.model, **sc.params))]
        npx = sc.image.size
        desc = f"{cfg} {sc.image.shape[0]}^2 {sc.model}, {iters} its"
    for r in runs:
        r.set_native_option("skip_uniform", a.skip_uniform)
    out = np.zeros(8)
    N.check(N.lib.lse_check_stats(N.dptr(out), 1))         # clear setup evaluations
    t1 = time.perf_counter()
    if cfg == "C4":
        from paper_1409_7474_b200.batch import TileBatch
        tb = TileBatch(runs)
        tb.advance(iters)
        tb.close()
    else:
        runs[0].advance(iters)
    N.check(N.lib.lse_check_stats(N.dptr(out), 1))
    t2 = time.perf_counter()
    fallbacks = sum(r.fallback_count() for r in runs)
    line = {
        "config": cfg, "workload": desc, "iterations": iters, "check_every": a.every,
        "skip_uniform": a.skip_uniform,
        "max_u_err_over_eps_u": out[0], "max_phi_err_over_eps_phi": out[1],
        "min_abs_u64": out[2], "min_abs_phi64": out[3],
        "bad_u_decisions": int(out[4]), "bad_phi_decisions": int(out[5]),
        "values_checked": int(out[6]), "pixel_iterations": npx * iters,
        "product_exact_fallbacks": int(fallbacks),
        "certified": bool(out[0] < 1 and out[1] < 1 and out[4] == 0 and out[5] == 0),
        "setup_s": round(t1 - t0, 1), "run_s": round(t2 - t1, 1),
    }
    s = json.dumps(line)
    print(s, flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
