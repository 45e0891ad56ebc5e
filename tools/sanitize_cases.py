"""Small runs of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck): tiled region (C5 crop), per-pixel region, edge,
zhang, a mixed batch, row strips (on-device emulation), 4 bands and the CV
baseline.  Each case checks its result against the oracle or the single run,
so a sanitizer-clean run is also a correct one.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys
import warnings

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402

import lse_oracle as O  # noqa: E402
import paper_1409_7474_b200 as L  # noqa: E402
from paper_1409_7474_b200 import scenes  # noqa: E402
from paper_1409_7474_b200.batch import TileBatch  # noqa: E402
from paper_1409_7474_b200.bands import BandEvolutionRun  # noqa: E402
from paper_1409_7474_b200.strips import run_local_strips  # noqa: E402


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def oracle_phi(img, poly, sign, model, iters, **kw):
    H, W = img.shape
    phi0 = O.rasterize_seeds(list(poly), sign, W, H)
    return O.run_fixed(img, phi0, O.OracleParams(model=model, max_iters=iters,
                                                 conv_check_every=iters + 1, **kw), iters).phi


def case_single(img, poly, sign, model, iters, **kw):
    p = params(model, max_iters=iters, conv_check_every=iters + 1, **kw)
    r = L.EvolutionRun(img, L.SeedSpec(polygons=tuple(poly), inside_sign=sign), p)
    r.advance(iters)
    ref = oracle_phi(img, poly, sign, model, iters, **kw)
    assert np.array_equal(r.state.phi, ref), f"{model}: differs from the oracle"
    return r


def main():
    which = sys.argv[1:] or ["tiled", "fine", "edge", "zhang", "batch", "strips", "bands", "cv"]
    sc = scenes.config5_crop(384, 12)
    if "tiled" in which:
        os.environ["LSE_FINE_MAX_PX"] = "0"
        case_single(sc.image.astype(np.float64), sc.polygons, sc.inside_sign, "region", 12,
                    dt=15.0, sigma2=1.5, ts_reg=9)
        os.environ.pop("LSE_FINE_MAX_PX")
        print("tiled region ok", flush=True)
    rng = np.random.default_rng(1)
    img = np.full((96, 80), 0.7)
    img[20:60, 15:50] = 0.25
    img = np.clip(img + 0.05 * rng.standard_normal(img.shape), 0, 1)
    poly = [np.array([[10.0, 12.0], [60.0, 12.0], [60.0, 70.0], [10.0, 70.0]])]
    if "fine" in which:
        case_single(img, poly, -1, "region", 10)
        print("per-pixel region ok", flush=True)
    if "edge" in which:
        case_single(img, poly, -1, "edge", 10)
        print("edge ok", flush=True)
    if "zhang" in which:
        case_single(img, poly, -1, "zhang", 10)
        print("zhang ok", flush=True)
    if "batch" in which:
        kinds = ["region", "edge", "zhang"]
        runs, single = [], []
        for k, m in enumerate(kinds):
            p = params(m, max_iters=8, conv_check_every=3, conv_window=2)
            seeds = L.SeedSpec(polygons=tuple(poly), inside_sign=-1)
            runs.append(L.EvolutionRun(img + 0.01 * k, seeds, p))
            single.append(L.EvolutionRun(img + 0.01 * k, seeds, p))
        os.environ["LSE_FINE_MAX_PX"] = "0"
        for r in single:
            r.advance(8)
        os.environ.pop("LSE_FINE_MAX_PX")
        TileBatch(runs).advance(8)
        for b, s in zip(runs, single):
            assert np.array_equal(b.state.phi, s.state.phi)
        print("batch ok", flush=True)
    if "strips" in which:
        p = params("region", max_iters=6)
        seeds = L.SeedSpec(polygons=tuple(poly), inside_sign=-1)
        ref = L.EvolutionRun(img, seeds, p)
        ref.advance(6)
        _, strips, _ = run_local_strips(img, seeds, p, 2, 6)
        phi = np.concatenate([s.own_phi() for s in strips])
        assert np.array_equal(phi, ref.state.phi)
        print("strips ok", flush=True)
    if "bands" in which:
        bands = np.stack([img, 1 - img, 0.5 * img, img ** 2])
        p = params("region", max_iters=6, conv_check_every=7)
        r = BandEvolutionRun(bands, L.SeedSpec(polygons=tuple(poly), inside_sign=-1), p)
        r.advance(6)
        print("bands ok", flush=True)
    if "cv" in which:
        p = params("cv", max_iters=6, conv_check_every=7)
        r = L.EvolutionRun(img, L.SeedSpec(polygons=tuple(poly), inside_sign=-1), p)
        r.advance(6)
        print("cv ok", flush=True)
    print("sanitize cases done")


if __name__ == "__main__":
    main()
