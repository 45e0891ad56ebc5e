"""Speculative fused iterations (lse_fast.cuh k_update_fused + k_spec_fix):
one pass per iteration computes the partition of b^n and b^{n+1} with
predicted coefficients, then the finalize checks the prediction and the
flagged pixels are decided exactly (or the update is redone).  The product
of every path must be the two-pass iteration's state bit for bit -- and the
reference's (oracle) -- whatever the prediction, the fix-list capacity, the
checkpoint cadence, convergence or the chunking of advance()."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from conftest import square

pytestmark = pytest.mark.gpu


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def tiled_env(mp):
    # small images: force the tiled kernels with unsplit units (the fused path)
    mp.setenv("LSE_FINE_MAX_PX", "0")
    mp.setenv("LSE_SPLIT_PARTS", "1")


def make_run(img, seeds, prm, chunks):
    r = L.EvolutionRun(img, seeds, prm)
    for n in chunks:
        r.advance(n)
    return r


def scene(h=300, w=530, seed=4):
    rng = np.random.default_rng(seed)
    img = np.full((h, w), 0.3)
    img[40:200, 60:300] = 0.72
    img[150:260, 350:500] = 0.65
    img = np.clip(img + 0.06 * rng.standard_normal((h, w)), 0, 1)
    return img, L.SeedSpec(polygons=(square(20, 20, w - 30, h - 25),), inside_sign=-1)


def same(a, b):
    sa, sb = a.state, b.state
    assert sa.iteration == sb.iteration and sa.converged == sb.converged
    assert sa.degenerate == sb.degenerate
    assert np.array_equal(sa.phi, sb.phi), np.abs(sa.phi - sb.phi).max()
    assert np.array_equal(a.mask(), b.mask())


@pytest.mark.parametrize("model", ["region", "zhang"])
def test_fused_matches_two_pass_and_oracle(model, monkeypatch):
    tiled_env(monkeypatch)
    img, seeds = scene()
    prm = params(model, max_iters=40, conv_check_every=41)
    fused = make_run(img, seeds, prm, [40])
    st = fused.spec_stats()
    assert st["enabled"] and st["fused"] == 39
    monkeypatch.setenv("LSE_FUSED", "0")
    plain = make_run(img, seeds, prm, [40])
    assert not plain.spec_stats()["enabled"]
    same(fused, plain)
    phi0 = O.rasterize_seeds(list(seeds.polygons), -1, img.shape[1], img.shape[0])
    ref = O.run_fixed(img, phi0, O.OracleParams(model=model, max_iters=40,
                                                conv_check_every=41), 40)
    assert np.array_equal(fused.state.phi, ref.phi)


def test_fused_convergence_and_chunks(monkeypatch):
    """Checkpoints decided inside the fused pass, convergence mid-chunk (the
    speculative b^{n+1} of the converged iteration is discarded), resumable
    advance: every chunking gives the two-pass result."""
    tiled_env(monkeypatch)
    img, seeds = scene(seed=9)
    prm = params("region", max_iters=400, conv_check_every=3, conv_window=2)
    runs = [make_run(img, seeds, prm, ch) for ch in ([400], [7, 1, 50, 400], [2] * 200)]
    monkeypatch.setenv("LSE_FUSED", "0")
    plain = make_run(img, seeds, prm, [400])
    assert plain.state.converged
    for r in runs:
        same(r, plain)


def test_forced_redo_path(monkeypatch):
    """A zero-capacity fix list: every speculative update with a flagged pixel
    is redone whole with the true coefficients."""
    tiled_env(monkeypatch)
    monkeypatch.setenv("LSE_FIX_CAP", "0")
    img, seeds = scene(seed=5)
    prm = params("region", max_iters=30, conv_check_every=5)
    r = make_run(img, seeds, prm, [30])
    st = r.spec_stats()
    assert st["redos"] >= 1 and st["fixes"] == 0
    monkeypatch.delenv("LSE_FIX_CAP")
    monkeypatch.setenv("LSE_FUSED", "0")
    same(r, make_run(img, seeds, prm, [30]))


def test_fix_list_used(monkeypatch):
    """Once the coefficients settle the prediction holds: most fused
    iterations are not redone and flagged pixels are decided from the list."""
    tiled_env(monkeypatch)
    img, seeds = scene(seed=6)
    prm = params("region", max_iters=80, conv_check_every=81)
    r = make_run(img, seeds, prm, [80])
    st = r.spec_stats()
    assert st["fused"] == 79 and st["redos"] < 8 and st["fixes"] > 0, st


def test_c5_crop_fused(monkeypatch):
    """C5 density crop (tiled; unsplit units, as at full size)."""
    monkeypatch.setenv("LSE_SPLIT_PARTS", "1")
    sc = scenes.config5_crop(2048, 60)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    prm = params("region", **sc.params)
    fused = make_run(sc.image, seeds, prm, [60])
    assert fused.spec_stats()["fused"] == 59
    monkeypatch.setenv("LSE_FUSED", "0")
    same(fused, make_run(sc.image, seeds, prm, [60]))


def test_degenerate_and_dense(monkeypatch):
    """A seed covering everything but a sliver (P nearly full, zero velocity
    reachable) and the dense pass (no uniform skip)."""
    tiled_env(monkeypatch)
    img, _ = scene(seed=7)
    seeds = L.SeedSpec(polygons=(square(1, 1, img.shape[1] - 2, img.shape[0] - 2),),
                       inside_sign=1)
    prm = params("region", max_iters=25, conv_check_every=4)
    a = L.EvolutionRun(img, seeds, prm)
    a.set_native_option("skip_uniform", 0)
    a.advance(25)
    monkeypatch.setenv("LSE_FUSED", "0")
    same(a, make_run(img, seeds, prm, [25]))


FUZZ_SHAPES = [(33, 31), (64, 257), (65, 264), (129, 70), (200, 520), (257, 263), (70, 1030),
               (1030, 70), (300, 777)]


@pytest.mark.parametrize("h,w", FUZZ_SHAPES)
@pytest.mark.parametrize("model,ts,f64", [("region", 9, False), ("region", 5, True),
                                          ("zhang", 7, False), ("region", 3, True)])
def test_fused_fuzz_geometry(h, w, model, ts, f64, monkeypatch):
    """Fused pass on every unit decomposition edge case (border-only images,
    partial word-rows, right tails / B1 packs), fp32 and float64 inputs (the
    exact data plane), random checkpoint cadence with convergence, chunked
    advance: identical to the two-pass iteration in every field, and to the
    oracle's trajectory."""
    tiled_env(monkeypatch)
    rng = np.random.default_rng(7 * h + 13 * w + ts)
    img = np.clip(0.3 + 0.4 * (rng.random((h, w)) > 0.6) + 0.05 * rng.standard_normal((h, w)),
                  0, 1)
    if not f64:
        img = img.astype(np.float32)
    y0, x0 = rng.integers(0, max(1, h // 3)), rng.integers(0, max(1, w // 3))
    y1, x1 = h - rng.integers(0, max(1, h // 3)), w - rng.integers(0, max(1, w // 3))
    poly = np.array([[x0 + 0.2, y0 + 0.2], [x1 - 0.2, y0 + 0.2], [x1 - 0.2, y1 - 0.2],
                     [x0 + 0.2, y1 - 0.2]])
    sign = 1 if rng.random() > 0.5 else -1
    if O.rasterize_seeds([poly], sign, w, h) is None:
        pytest.skip("degenerate seed for this draw")
    cce = int(rng.integers(2, 6))
    prm = params(model, ts_reg=ts, max_iters=60, conv_check_every=cce, conv_window=2)
    seeds = L.SeedSpec(polygons=(poly,), inside_sign=sign)
    chunks = [int(c) for c in rng.integers(1, 9, size=12)]
    fused = make_run(img, seeds, prm, chunks)
    monkeypatch.setenv("LSE_FUSED", "0")
    plain = make_run(img, seeds, prm, chunks)
    same(fused, plain)
    it = fused.state.iteration
    phi0 = O.rasterize_seeds([poly], sign, w, h)
    ref = O.run_fixed(np.asarray(img, dtype=np.float64), phi0,
                      O.OracleParams(model=model, ts_reg=ts, max_iters=it,
                                     conv_check_every=it + 1), it)
    assert np.array_equal(fused.state.phi, ref.phi)
