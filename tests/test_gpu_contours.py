"""Zero-level contours on the device (marching squares kernel + native
segment assembly) against the oracle restatement of the reference's
extract_contours (engine.py:280-294): same contours, same order, same points,
bit for bit; and the checkpoint trace of EvolutionRun (engine.py:214-238)."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L
from conftest import square, two_region

pytestmark = pytest.mark.gpu


def same(a, b):
    assert len(a) == len(b), (len(a), len(b))
    for x, y in zip(a, b):
        assert x.shape == y.shape and x.dtype == np.float64
        assert np.array_equal(x, y)


def fields():
    rng = np.random.default_rng(7)
    yield rng.standard_normal((37, 53))                        # many small loops, open ones
    yield rng.integers(-1, 2, (64, 48)).astype(np.float64)     # exact zeros everywhere
    yield np.where(rng.random((40, 40)) < 0.5, 1.0, -1.0)      # saddles (cases 6 / 9)
    yy, xx = np.mgrid[0:300, 0:200]
    yield np.sin(xx / 9.0) * np.cos(yy / 13.0) - 0.1          # a smooth lattice of loops
    f = rng.standard_normal((50, 50))
    f[rng.random((50, 50)) < 0.05] = np.nan                    # NaN corners skip squares
    yield f
    yield rng.standard_normal((2, 2))
    yield rng.standard_normal((1, 17))                          # no squares
    yield rng.standard_normal((23, 1))
    n, r = 64, 20.0
    yy, xx = np.mgrid[0:n, 0:n]
    yield np.hypot(xx - 31.5, yy - 31.5) - r


def test_extract_contours_matches_oracle():
    for k, phi in enumerate(fields()):
        same(L.extract_contours(phi), O.extract_contours(phi))


def test_reference_contour_tests():                   # tests/test_engine.py:202-228
    assert L.extract_contours(np.ones((8, 8))) == []
    phi = np.ones((32, 32))
    phi[8:20, 10:24] = -1.0
    cs = L.extract_contours(phi)
    assert len(cs) == 1 and np.allclose(cs[0][0], cs[0][-1])


def test_large_field_matches_oracle():
    rng = np.random.default_rng(3)
    low = rng.standard_normal((65, 65))
    phi = np.kron(low, np.ones((16, 16)))[:1031, :1000] + 0.01 * rng.standard_normal((1031, 1000))
    same(L.extract_contours(phi), O.extract_contours(phi))
    phi32 = phi.astype(np.float32)             # coerced to float64 like np.asarray(phi, float64)
    same(L.extract_contours(phi32), O.extract_contours(phi32.astype(np.float64)))


def _params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(model, **kw)


def _oracle_params(p):
    mp = p.model_params
    return O.OracleParams(model=p.model.value, dt=p.dt, sigma2=p.sigma2, ts_reg=p.ts_reg,
                          reinit_period=p.reinit_period, reg_period=p.reg_period,
                          max_iters=p.max_iters, conv_check_every=p.conv_check_every,
                          conv_window=p.conv_window, sigma1=mp.sigma1, ts_pre=mp.ts_pre,
                          edge_gain=mp.edge_gain, nu=mp.nu, mu=mp.mu)


@pytest.mark.parametrize("model", ["region", "edge", "zhang"])
def test_trace_matches_oracle(model):
    img, _ = two_region(96, 30, 70)
    img = img + 0.05 * np.random.default_rng(1).standard_normal(img.shape)
    seeds = L.SeedSpec(polygons=(square(10, 12, 84, 80),), inside_sign=-1)
    p = _params(L.ModelKind(model), max_iters=60, conv_check_every=7)
    r = L.EvolutionRun(img, seeds, p, trace=True)
    phi0 = O.rasterize_seeds([q for q in seeds.polygons], seeds.inside_sign, 96, 96)
    o = O.OracleRun(img, phi0, _oracle_params(p), trace=True)
    r.advance(25)
    r.advance(3)
    r.advance(100)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        o.advance(128)
    assert r.state.iteration == o.iteration
    assert [n for n, _ in r.trace] == [n for n, _ in o.trace]
    for (_, a), (_, b) in zip(r.trace, o.trace):
        same(a, b)
    same(r.contours(), O.extract_contours(o.phi))
    res = L.run(img, seeds, p, trace=True)
    assert isinstance(res.trace, tuple) and len(res.trace) == len(o.trace)
    for (n, a), (m, b) in zip(res.trace, o.trace):
        assert n == m
        same(a, b)


def test_trace_stops_at_convergence():
    img, _ = two_region(64, 20, 44)
    seeds = L.SeedSpec(polygons=(square(8, 8, 56, 56),), inside_sign=-1)
    p = _params(L.ModelKind.REGION, max_iters=500, conv_check_every=5, conv_window=3)
    r = L.EvolutionRun(img, seeds, p, trace=True)
    r.advance(500)
    assert r.converged
    phi0 = O.rasterize_seeds([q for q in seeds.polygons], -1, 64, 64)
    o = O.OracleRun(img, phi0, _oracle_params(p), trace=True).advance(500)
    assert o.converged and [n for n, _ in r.trace] == [n for n, _ in o.trace]
    same(r.trace[-1][1], o.trace[-1][1])


def test_band_run_trace_equals_single_band():
    from paper_1409_7474_b200.bands import BandEvolutionRun
    img, _ = two_region(80, 25, 55)
    seeds = L.SeedSpec(polygons=(square(10, 10, 70, 70),), inside_sign=-1)
    p = _params(L.ModelKind.REGION, max_iters=30, conv_check_every=10)
    a = L.EvolutionRun(img, seeds, p, trace=True)
    b = BandEvolutionRun(img[None], seeds, p, trace=True)
    a.advance(30)
    b.advance(30)
    assert [n for n, _ in a.trace] == [n for n, _ in b.trace] == [0, 10, 20, 30]
    for (_, x), (_, y) in zip(a.trace, b.trace):
        same(x, y)
