"""Resident kernel of small images (lse_resident.cuh): a whole advance() call
is one launch, iterations separated by cluster / grid barriers.  Its state
must equal the per-iteration kernels' (LSE_RESIDENT=0) and the reference's
(goldens / oracle) bit for bit -- for both barrier kinds, every model of the
binary-state path, checkpoints / convergence inside the kernel and every
chunking of advance()."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from conftest import load_golden, square

pytestmark = pytest.mark.gpu


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def make_run(img, seeds, prm, chunks):
    r = L.EvolutionRun(img, seeds, prm)
    for n in chunks:
        r.advance(n)
    return r


def scene(h=200, w=230, seed=4):
    rng = np.random.default_rng(seed)
    img = np.full((h, w), 0.3)
    img[40:150, 60:170] = 0.72
    img[120:190, 150:220] = 0.65
    img = np.clip(img + 0.06 * rng.standard_normal((h, w)), 0, 1)
    return img, L.SeedSpec(polygons=(square(20, 20, w - 30, h - 25),), inside_sign=-1)


def same(a, b):
    sa, sb = a.state, b.state
    assert sa.iteration == sb.iteration and sa.converged == sb.converged
    assert sa.degenerate == sb.degenerate
    assert np.array_equal(sa.phi, sb.phi), np.abs(sa.phi - sb.phi).max()
    assert np.array_equal(a.mask(), b.mask())


MODES = [("1", False), ("2", True)]      # LSE_RESIDENT value, grid barrier?


@pytest.mark.parametrize("mode,grid", MODES)
@pytest.mark.parametrize("model", ["region", "zhang", "edge"])
def test_resident_matches_launch_chain_and_oracle(model, mode, grid, monkeypatch):
    img, seeds = scene()
    kw = dict(nu=-1.0) if model == "zhang" else {}
    prm = params(model, max_iters=40, conv_check_every=7, conv_window=50, **kw)
    monkeypatch.setenv("LSE_RESIDENT", mode)
    res = make_run(img, seeds, prm, [40])
    st = res.resident_stats()
    assert st["enabled"] and st["grid"] == grid and st["calls"] == 1, st
    monkeypatch.setenv("LSE_RESIDENT", "0")
    plain = make_run(img, seeds, prm, [40])
    assert not plain.resident_stats()["enabled"]
    same(res, plain)
    assert res.state.iteration == 40
    phi0 = O.rasterize_seeds(list(seeds.polygons), -1, img.shape[1], img.shape[0])
    op = O.OracleParams(model=model, max_iters=40, conv_check_every=7, conv_window=50, **kw)
    ref = O.run_fixed(img, phi0, op, 40)
    assert np.array_equal(res.state.phi, ref.phi)


@pytest.mark.parametrize("mode,grid", MODES)
def test_resident_convergence_and_chunks(mode, grid, monkeypatch):
    """Convergence decided inside the kernel (the state stays at the converged
    iteration), resumable advance: every chunking gives the same run."""
    img, seeds = scene(seed=9)
    prm = params("region", max_iters=600, conv_check_every=3, conv_window=2)
    monkeypatch.setenv("LSE_RESIDENT", mode)
    runs = [make_run(img, seeds, prm, ch) for ch in ([600], [7, 1, 50, 600], [2] * 300, [1] * 40 + [600])]
    assert all(r.resident_stats()["enabled"] for r in runs)
    monkeypatch.setenv("LSE_RESIDENT", "0")
    plain = make_run(img, seeds, prm, [600])
    assert plain.state.converged and plain.state.iteration < 600
    for r in runs:
        same(r, plain)


@pytest.mark.parametrize("mode,grid", MODES)
def test_resident_edge_convergence(mode, grid, monkeypatch):
    sc = scenes.config2()
    img = sc.image[200:520, 300:700]
    seeds = L.SeedSpec(polygons=(square(30, 30, 370, 290),), inside_sign=sc.inside_sign)
    prm = params("edge", **{**sc.params, "max_iters": 300, "conv_check_every": 5, "conv_window": 2})
    img = np.ascontiguousarray(img)
    monkeypatch.setenv("LSE_RESIDENT", mode)
    res = make_run(img, seeds, prm, [120, 180])
    assert res.resident_stats()["enabled"]
    monkeypatch.setenv("LSE_RESIDENT", "0")
    plain = make_run(img, seeds, prm, [300])
    same(res, plain)


@pytest.mark.parametrize("mode,grid", MODES)
def test_c1_golden(mode, grid, monkeypatch):
    """BASELINE C1 (256^2 region, dt 100, 200 iterations): the reference's phi
    (SHA-256 of the float64 bytes), one cluster of 16 CTAs."""
    from test_gpu_parity import params_from, sha
    g = load_golden("traj_C1")
    sc = scenes.config1()
    monkeypatch.setenv("LSE_RESIDENT", mode)
    r = L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),
                       params_from(g))
    r.advance(sc.iters)
    st = r.resident_stats()
    assert st["enabled"] and st["grid"] == grid
    if not grid:
        assert st["ctas"] == 16
    assert r.state.iteration == sc.iters
    phi = r.state.phi
    assert np.array_equal(np.packbits(phi > 0), g[f"mask_{sc.iters}"])
    assert sha(phi) == str(g[f"sha_{sc.iters}"])


@pytest.mark.parametrize("shape", [(33, 40), (64, 8), (31, 257), (256, 256), (97, 300), (400, 130)])
@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_shapes_and_radii(shape, R, monkeypatch):
    """Ragged sizes (partial column blocks, partial word-rows, images narrower
    than the stencil) and every template radius, both barrier kinds."""
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w + R)
    img = np.clip(0.3 + 0.4 * (rng.random((h, w)) > 0.6) + 0.05 * rng.standard_normal((h, w)), 0, 1)
    seeds = L.SeedSpec(polygons=(square(2, 2, max(4, w - 3), max(4, h - 3)),), inside_sign=-1)
    prm = params("region", max_iters=25, conv_check_every=4, conv_window=30, ts_reg=2 * R + 1)
    out = []
    for mode in ("1", "2", "0"):
        monkeypatch.setenv("LSE_RESIDENT", mode)
        out.append(make_run(img, seeds, prm, [25]))
    assert out[0].resident_stats()["enabled"] and out[1].resident_stats()["grid"]
    same(out[0], out[2])
    same(out[1], out[2])


def test_degenerate_and_float32_image(monkeypatch):
    """A constant image (zero velocity from the first update: the sticky
    degenerate flag) and a float32 image whose fp32 plane is exact."""
    flat = np.full((64, 72), 0.5)
    seeds = L.SeedSpec(polygons=(square(0, 0, 72, 30),), inside_sign=-1)
    prm = params("region", max_iters=10, conv_check_every=3, conv_window=20)
    img32, seeds32 = scene(seed=11)
    img32 = img32.astype(np.float32)
    for image, sd, degenerate in ((flat, seeds, True), (img32, seeds32, False)):
        out = []
        for mode in ("1", "0"):
            monkeypatch.setenv("LSE_RESIDENT", mode)
            out.append(make_run(image, sd, prm, [4, 6]))
        assert out[0].resident_stats()["calls"] == 2
        same(out[0], out[1])
        assert out[0].state.degenerate == degenerate


def test_c2_golden_several_tasks_per_warp():
    """BASELINE C2 (1024^2 edge, 500 iterations): 4096 warp tasks on a
    cooperative grid, two per warp; the reference's phi (SHA-256)."""
    from test_gpu_parity import params_from, sha
    g = load_golden("traj_C2")
    sc = scenes.config2()
    r = L.EvolutionRun(sc.image, L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign),
                       params_from(g))
    for n in (130, 1, sc.iters):
        r.advance(n)
    st = r.resident_stats()
    assert st["enabled"] and st["grid"] and st["tasks_per_warp"] >= 2, st
    assert r.state.iteration == sc.iters
    assert sha(r.state.phi) == str(g[f"sha_{sc.iters}"])


@pytest.mark.parametrize("shape", [(700, 900), (1100, 1300)])
@pytest.mark.parametrize("model", ["edge", "region", "zhang"])
def test_large_matches_launch_chain(shape, model, monkeypatch):
    """Runs beyond the per-pixel size range (2 and 3 tasks per warp on a full
    cooperative grid; region runs keep phi of every task across the
    coefficient barrier), convergence checkpoints included -- against the
    tiled kernels (the speculative fused pass for region / zhang)."""
    h, w = shape
    rng = np.random.default_rng(h + w)
    img = np.full((h, w), 0.35)
    img[h // 4: 3 * h // 4, w // 3: 2 * w // 3] = 0.7
    img = np.clip(img + 0.03 * rng.standard_normal((h, w)), 0, 1)
    seeds = L.SeedSpec(polygons=(square(40, 40, w - 50, h - 60),), inside_sign=-1)
    prm = params(model, max_iters=60, conv_check_every=6, conv_window=40)
    res = make_run(img, seeds, prm, [25, 35])
    st = res.resident_stats()
    assert st["enabled"] and st["grid"] and st["tasks_per_warp"] >= 2, st
    monkeypatch.setenv("LSE_RESIDENT", "0")
    same(res, make_run(img, seeds, prm, [60]))


def test_size_limit(monkeypatch):
    """Beyond three tasks per warp of the grid (and above LSE_RESIDENT_MAX_PX)
    the tiled kernels run."""
    img = np.full((1700, 1500), 0.4)
    img[300:900, 200:1000] = 0.8
    seeds = L.SeedSpec(polygons=(square(50, 50, 1400, 1600),), inside_sign=-1)
    r = L.EvolutionRun(img, seeds, params("region", max_iters=3))
    assert not r.resident_stats()["enabled"]
    monkeypatch.setenv("LSE_RESIDENT_MAX_PX", "10000")
    small, sd = scene()
    assert not L.EvolutionRun(small, sd, params("region", max_iters=3)).resident_stats()["enabled"]
