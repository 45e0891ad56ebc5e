"""Multi-band region model on the device: K = 1 equals the
single-band region path (and so the reference), K = 4 equals the oracle's
restatement bit for bit."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from paper_1409_7474_b200.bands import BandEvolutionRun
from conftest import load_golden, square

pytestmark = pytest.mark.gpu


def params(**kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.REGION, **kw)


def oracle(bands, phi0, prm, iters):
    op = O.OracleParams(model="region", dt=prm.dt, sigma2=prm.sigma2, ts_reg=prm.ts_reg,
                        max_iters=prm.max_iters, conv_check_every=prm.conv_check_every,
                        conv_window=prm.conv_window)
    r = O.OracleRun(np.asarray(bands, dtype=np.float64), phi0, op)
    r.advance(iters)
    return r


def test_one_band_is_the_reference_region_trajectory():
    g = load_golden("traj_region_small")
    img = g["image"]
    seeds = L.SeedSpec(polygons=tuple(q for q in g["poly"]), inside_sign=int(g["inside_sign"]))
    r = BandEvolutionRun(img[None], seeds, params(max_iters=25))
    for it in g["iters_recorded"]:
        r.advance(int(it) - r.state.iteration)
        assert np.array_equal(r.state.phi, g[f"phi_{it}"]), it


@pytest.mark.parametrize("k", [2, 4])
def test_bands_match_oracle(k):
    rng = np.random.default_rng(k)
    h, w = 90, 75
    base = np.array([0.25, 0.30, 0.28, 0.45])[:k]
    fg = np.array([0.60, 0.62, 0.65, 0.35])[:k]
    bands = base[:, None, None] + 0.05 * rng.standard_normal((k, h, w))
    bands[:, 20:60, 15:55] = fg[:, None, None] + 0.04 * rng.standard_normal((k, 40, 40))
    bands = np.clip(bands, 0, 1)
    seeds = L.SeedSpec(polygons=(square(8, 10, 66, 80),), inside_sign=-1)
    prm = params(max_iters=200, conv_check_every=5, conv_window=2)
    r = BandEvolutionRun(bands, seeds, prm)
    r.advance(200)
    phi0 = O.rasterize_seeds([square(8, 10, 66, 80)], -1, w, h)
    ref = oracle(bands, phi0, prm, 200)
    assert r.state.iteration == ref.iteration and r.converged == ref.converged
    assert np.array_equal(r.state.phi, ref.phi)


def test_c3_crop_checkerboard_matches_oracle():
    sc = scenes.config3(512, 40)
    prm = params(**sc.params)
    r = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r.advance(40)
    ref = oracle(sc.image, sc.extra["signs"].astype(np.float64), prm, 40)
    assert np.array_equal(r.state.phi, ref.phi)
    assert np.array_equal(r.mask(), ref.phi > 0)


def test_band_runs_refuse_the_generic_path():
    bands = np.random.default_rng(0).random((2, 40, 40))
    seeds = L.SeedSpec(polygons=(square(5, 5, 30, 30),))
    with pytest.raises(RuntimeError):
        BandEvolutionRun(bands, seeds, params(reinit_period=2))


def test_peak_pass_reuse_is_exact(monkeypatch):
    """Once the partition stops moving (C3's checkerboard settles within ~40
    iterations) the band means, D and max|D| are bit-identical and the peak
    pass is reused; the trajectory equals the recomputed one and the oracle."""
    sc = scenes.config3(512, 90)
    prm = params(**sc.params)
    r = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r.advance(90)
    st = r.band_stats()
    assert st["enabled"] and st["reused"] > 10
    monkeypatch.setenv("LSE_BAND_REUSE", "0")
    r0 = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r0.advance(90)
    assert r0.band_stats() == dict(reused=0, enabled=False)
    assert np.array_equal(r.state.phi, r0.state.phi)
    ref = oracle(sc.image, sc.extra["signs"].astype(np.float64), prm, 90)
    assert np.array_equal(r.state.phi, ref.phi)


def test_peak_pass_reuse_with_checkpoints():
    """Reuse across checkpoint / convergence bookkeeping: the convergence
    iteration and the final state equal the oracle's."""
    sc = scenes.config3(256, 200)
    prm = params(**dict(sc.params, max_iters=200, conv_check_every=7, conv_window=3))
    r = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r.advance(200)
    ref = oracle(sc.image, sc.extra["signs"].astype(np.float64), prm, 200)
    assert r.state.iteration == ref.iteration and r.converged == ref.converged
    assert np.array_equal(r.state.phi, ref.phi)
