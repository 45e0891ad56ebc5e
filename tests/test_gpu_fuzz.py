"""Randomized geometry sweep: image sizes across the unit decomposition's
edge cases (narrower than a lane group, shorter than a word-row, right tails,
partial word-rows, split-warp and full units, both models, odd templates),
every trajectory compared bit for bit with the oracle."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L

pytestmark = pytest.mark.gpu

CASES = [(h, w) for h, w in [(3, 5), (7, 9), (31, 33), (32, 32), (33, 31), (40, 8), (8, 40),
                             (64, 257), (65, 264), (96, 300), (129, 70), (200, 520),
                             (257, 263), (70, 1030), (1030, 70)]]


@pytest.mark.parametrize("h,w", CASES)
@pytest.mark.parametrize("model,ts", [("region", 9), ("edge", 9), ("region", 5), ("zhang", 7)])
def test_random_geometry_matches_oracle(h, w, model, ts):
    rng = np.random.default_rng(h * 1000 + w + ts)
    img = np.clip(0.3 + 0.4 * (rng.random((h, w)) > 0.5) + 0.05 * rng.standard_normal((h, w)),
                  0, 1)
    y0, x0 = rng.integers(0, max(1, h // 3)), rng.integers(0, max(1, w // 3))
    y1, x1 = h - rng.integers(0, max(1, h // 3)), w - rng.integers(0, max(1, w // 3))
    poly = np.array([[x0 + 0.2, y0 + 0.2], [x1 - 0.2, y0 + 0.2], [x1 - 0.2, y1 - 0.2],
                     [x0 + 0.2, y1 - 0.2]])
    sign = 1 if rng.random() > 0.5 else -1
    phi0 = O.rasterize_seeds([poly], sign, w, h)
    if phi0 is None:
        pytest.skip("degenerate seed for this draw")
    iters = 12
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        p = L.default_params(L.ModelKind.from_name(model), ts_reg=ts, max_iters=iters,
                             conv_check_every=iters + 1)
    r = L.EvolutionRun(img, L.SeedSpec(polygons=(poly,), inside_sign=sign), p)
    r.advance(iters)
    op = O.OracleParams(model=model, ts_reg=ts, max_iters=iters, conv_check_every=iters + 1)
    ref = O.run_fixed(img, phi0, op, iters)
    assert np.array_equal(r.state.phi, ref.phi), np.abs(r.state.phi - ref.phi).max()


# Every forced work decomposition (the tiled kernels' split-warp row parts x
# border row parts, or the per-pixel kernels; lse_api.cu reads LSE_FINE_MAX_PX,
# LSE_SPLIT_PARTS and LSE_BORDER_Q when a run is created) gives the oracle's
# trajectory bit for bit.
@pytest.mark.parametrize("h,w", [(96, 300), (200, 520), (257, 263), (300, 1100)])
@pytest.mark.parametrize("split,bq", [(1, 4), (2, 8), (4, 4), (4, 16), (1, 16), ("fine", 0)])
@pytest.mark.parametrize("model", ["region", "edge"])
def test_forced_decomposition_matches_oracle(h, w, split, bq, model, monkeypatch):
    if split == "fine":
        monkeypatch.setenv("LSE_FINE_MAX_PX", str(1 << 30))
        split, bq = 1, 4
    else:
        monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    monkeypatch.setenv("LSE_SPLIT_PARTS", str(split))
    monkeypatch.setenv("LSE_BORDER_Q", str(bq))
    rng = np.random.default_rng(h * 7 + w + bq)
    img = np.clip(0.3 + 0.4 * (rng.random((h, w)) > 0.6) + 0.05 * rng.standard_normal((h, w)),
                  0, 1)
    poly = np.array([[w * 0.1, h * 0.15], [w * 0.85, h * 0.1], [w * 0.9, h * 0.8],
                     [w * 0.2, h * 0.9]])
    sign = -1 if model == "edge" else 1
    phi0 = O.rasterize_seeds([poly], sign, w, h)
    iters = 15
    p = L.default_params(L.ModelKind.from_name(model), max_iters=iters,
                         conv_check_every=iters + 1)
    r = L.EvolutionRun(img, L.SeedSpec(polygons=(poly,), inside_sign=sign), p)
    r.advance(iters)
    op = O.OracleParams(model=model, max_iters=iters, conv_check_every=iters + 1)
    ref = O.run_fixed(img, phi0, op, iters)
    assert np.array_equal(r.state.phi, ref.phi), np.abs(r.state.phi - ref.phi).max()


# The random-geometry sweep above runs the per-pixel kernels (small images);
# the same sweep through the tiled kernels.
@pytest.mark.parametrize("h,w", CASES)
@pytest.mark.parametrize("model,ts", [("region", 9), ("edge", 9), ("zhang", 7)])
def test_random_geometry_tiled_matches_oracle(h, w, model, ts, monkeypatch):
    monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    test_random_geometry_matches_oracle(h, w, model, ts)


# Sizes either side of the per-pixel / tiled switch (450 000 pixels) and
# extreme aspect ratios, through the default decomposition choice.
@pytest.mark.parametrize("h,w", [(600, 700), (700, 700), (90, 5100), (5100, 90), (33, 16000)])
@pytest.mark.parametrize("model", ["region", "edge"])
def test_switch_sizes_match_oracle(h, w, model):
    rng = np.random.default_rng(h + 7 * w)
    img = np.clip(0.3 + 0.4 * (rng.random((h, w)) > 0.7) + 0.05 * rng.standard_normal((h, w)),
                  0, 1)
    poly = np.array([[w * 0.05, h * 0.1], [w * 0.9, h * 0.05], [w * 0.95, h * 0.85],
                     [w * 0.1, h * 0.95]])
    sign = -1 if model == "edge" else 1
    phi0 = O.rasterize_seeds([poly], sign, w, h)
    iters = 10
    p = L.default_params(L.ModelKind.from_name(model), max_iters=iters,
                         conv_check_every=iters + 1)
    r = L.EvolutionRun(img, L.SeedSpec(polygons=(poly,), inside_sign=sign), p)
    r.advance(iters)
    op = O.OracleParams(model=model, max_iters=iters, conv_check_every=iters + 1)
    ref = O.run_fixed(img, phi0, op, iters)
    assert np.array_equal(r.state.phi, ref.phi), np.abs(r.state.phi - ref.phi).max()
