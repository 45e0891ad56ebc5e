"""Parity at the BASELINE.json sizes (SURVEY.md section 8d "Parity runs").

Each test runs a BASELINE config (or the crop section 8d names) on the device
through the package API and compares phi with the C restatement of the
reference loop (oracle/lse_oracle.c, itself pinned bit-exact to the
reference's goldens by tests/test_oracle_c.py) on identical float32-exact
inputs:

* C5: a 4096^2 crop at the C5 object density for the full 500 iterations,
  and the full 32768^2 scene for 3 iterations;
* C4: tiles 0-15 (1024^2 8-bit RGB, luma decoded on the device), region /
  edge alternating, 300 iterations, advanced as one batch;
* C3: 4096^2 x 4 bands, +-1 checkerboard of 64^2 cells, 200 iterations.

Bar: phi bit-identical (every sign decision equals the fp64 reference's),
which implies north_star's 1e-4 relative phi / 0.01 % mask bar.
"""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import lse_oracle_c as OC
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes

pytestmark = pytest.mark.gpu


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def oracle_params(prm, iters):
    mp = prm.model_params
    return O.OracleParams(model=prm.model.value, dt=prm.dt, sigma2=prm.sigma2,
                          ts_reg=prm.ts_reg, max_iters=iters, conv_check_every=iters + 1,
                          sigma1=mp.sigma1, ts_pre=mp.ts_pre, edge_gain=mp.edge_gain)


def assert_phi_equal(got, want, what):
    if np.array_equal(got, want):
        return
    rng = float(want.max() - want.min()) or 1.0
    err = float(np.abs(got - want).max()) / rng
    mism = float(np.count_nonzero((got > 0) != (want > 0))) / want.size
    raise AssertionError(f"{what}: phi not bit-identical (max |dphi| / range = {err:.3e}, "
                         f"mask disagreement {100 * mism:.5f} %)")


def host_ram_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2 ** 30
    except Exception:
        return 0.0


def test_c5_crop_4096_full_500_iterations():
    size, iters = 4096, 500
    sc = scenes.config5_crop(size, iters)
    prm = params("region", **sc.params)
    r = L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),
                       prm)
    r.set_native_option("skip_uniform", 0)              # the dense pass of the headline
    r.advance(iters)
    assert r.state.iteration == iters
    phi = r.state.phi
    phi0 = O.rasterize_seeds(list(sc.polygons), sc.inside_sign, size, size)
    ref = OC.COracleRun(sc.image.astype(np.float64), phi0, oracle_params(prm, iters),
                        O.gaussian_weights)
    ref.advance(iters)
    assert ref.iteration == iters
    assert_phi_equal(phi, ref.phi, "C5 4096^2 crop x 500")


def test_c5_full_scene_3_iterations():
    size, iters = 32768, 3
    if host_ram_gb() < 90:
        pytest.skip(f"needs ~90 GB of host RAM for the oracle ({host_ram_gb():.0f} GB free)")
    sc = scenes.config5(size=size, iters=iters)
    prm = params("region", **sc.params)
    r = L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),
                       prm)
    r.set_native_option("skip_uniform", 0)
    r.advance(iters)
    assert r.state.iteration == iters
    phi = r.state.phi
    del r
    img64 = sc.image.astype(np.float64)
    del sc.image
    phi0 = O.rasterize_seeds(list(sc.polygons), sc.inside_sign, size, size)
    ref = OC.COracleRun(img64, phi0, oracle_params(prm, iters), O.gaussian_weights)
    del img64, phi0
    ref.advance(iters)
    assert ref.iteration == iters
    # compare in row blocks (two 8.6 GB fields)
    for y in range(0, size, 4096):
        assert_phi_equal(phi[y:y + 4096], ref.phi[y:y + 4096], f"C5 32768^2 rows {y}..")


def test_c4_tiles_0_15_batched_match_oracle():
    from paper_1409_7474_b200.batch import TileBatch, _tile_run
    n, size, iters = 16, 1024, 300
    sc = [scenes.config4_tile(k, size, iters) for k in range(n)]
    prm = [params(s.model, **s.params) for s in sc]
    runs = [_tile_run(s.image, L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign), p)
            for s, p in zip(sc, prm)]
    for r in runs:
        r.set_native_option("skip_uniform", 0)
    tb = TileBatch(runs)
    tb.advance(iters)
    tb.close()
    for k, (s, p, r) in enumerate(zip(sc, prm, runs)):
        assert r.state.iteration == iters
        phi0 = O.rasterize_seeds(list(s.polygons), s.inside_sign, size, size)
        ref = OC.COracleRun(scenes.luma(s.image), phi0, oracle_params(p, iters),
                            O.gaussian_weights)
        ref.advance(iters)
        assert_phi_equal(r.state.phi, ref.phi, f"C4 tile {k} ({s.model})")
        want = (ref.phi > 0) if s.inside_sign > 0 else (ref.phi <= 0)
        assert np.array_equal(r.mask(), want)


def test_c3_4096_bands_200_iterations_match_restatement():
    from paper_1409_7474_b200.bands import BandEvolutionRun
    size, iters = 4096, 200
    sc = scenes.config3(size, iters)
    prm = params("region", **sc.params)
    r = BandEvolutionRun(sc.image, sc.extra["signs"], prm)
    r.set_native_option("skip_uniform", 0)
    r.advance(iters)
    assert r.state.iteration == iters
    ref = OC.COracleRun(sc.image.astype(np.float64), sc.extra["signs"].astype(np.float64),
                        oracle_params(prm, iters), O.gaussian_weights)
    ref.advance(iters)
    assert ref.iteration == iters
    assert_phi_equal(r.state.phi, ref.phi, "C3 4096^2 x 4 bands x 200")
