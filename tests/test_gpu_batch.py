"""Batched tiles: many equal-size tiles advanced with one launch
per kernel per iteration must evolve exactly as each tile alone; 8-bit RGB
tiles are decoded on the device to the reference loader's luma."""
import warnings

import numpy as np
import pytest

import lse_oracle as O
import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from paper_1409_7474_b200.batch import TileBatch, _tile_run, run_tiles, run_tiles_sharded
from conftest import load_golden, square, two_region

pytestmark = pytest.mark.gpu


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def tile(k, h=100, w=80):
    rng = np.random.default_rng(100 + k)
    img = np.full((h, w), 0.2 + 0.05 * k)
    img[20 + k:70, 15:60 - k] = 0.75
    return np.clip(img + 0.06 * rng.standard_normal((h, w)), 0, 1)


def check_same(batch_runs, single_runs):
    for b, s in zip(batch_runs, single_runs):
        sb, ss = b.state, s.state
        assert sb.iteration == ss.iteration and sb.converged == ss.converged
        assert sb.degenerate == ss.degenerate
        assert np.array_equal(sb.phi, ss.phi)
        assert np.array_equal(b.mask(), s.mask())


def mixed_case(h):
    kinds = ["region", "edge", "zhang", "region", "edge"]
    kw = dict(max_iters=60, conv_check_every=4, conv_window=2)
    seeds = [L.SeedSpec(polygons=(square(6, 8, 70, h - 10),), inside_sign=(-1) ** k)
             for k in range(len(kinds))]
    prm = [params(m, **kw) for m in kinds]
    imgs = [tile(k, h) for k in range(len(kinds))]
    return imgs, seeds, prm


@pytest.mark.parametrize("h", [100, 96])
def test_mixed_models_match_single_runs(h, monkeypatch):
    """A batched tile equals the same tile run alone on the tiled kernels
    (LSE_FINE_MAX_PX=0: the lone tile groups its partials as the batch does)."""
    imgs, seeds, prm = mixed_case(h)
    monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    for r in single:
        r.advance(60)
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    TileBatch(batch).advance(60)
    check_same(batch, single)


@pytest.mark.parametrize("h", [100, 96])
def test_mixed_models_match_single_runs_across_paths(h):
    """Cross-path check: the lone tiles run the per-pixel kernels (their c+/c-
    partials are grouped per CTA, the batch's per tiled unit); the
    trajectories still agree here."""
    imgs, seeds, prm = mixed_case(h)
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    for r in single:
        r.advance(60)
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    TileBatch(batch).advance(60)
    check_same(batch, single)


def test_two_stage_batched_finalize_matches_single_runs(monkeypatch):
    """LSE_ONESTAGE_MAX_PARTS=0 forces the two-stage per-tile finalize
    (k_finalize_stage1_tiles + k_finalize_run_tiles) that tiles of >= ~3000^2
    take; a batched tile still equals the tile alone (tiled path, two-stage)."""
    imgs, seeds, prm = mixed_case(100)
    monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    monkeypatch.setenv("LSE_ONESTAGE_MAX_PARTS", "0")
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    for r in single:
        r.advance(60)
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    TileBatch(batch).advance(60)
    check_same(batch, single)
    # and the two-stage result equals the default (one-stage) one
    monkeypatch.setenv("LSE_ONESTAGE_MAX_PARTS", "768")
    one = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    TileBatch(one).advance(60)
    for a, b in zip(one, batch):
        assert np.array_equal(a.mask(), b.mask())


@pytest.mark.parametrize("h,stages", [(100, "one"), (96, "one"), (100, "two")])
def test_fused_batch_matches_single_runs(h, stages, monkeypatch):
    """The opt-in batched speculative pass (LSE_FUSED_BATCH=1): mixed region /
    edge / zhang tiles converging at different iterations, chunked advance,
    the one- and two-stage per-tile finalize -- every tile equals the tile
    alone, bit for bit."""
    imgs, seeds, prm = mixed_case(h)
    monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    if stages == "two":
        monkeypatch.setenv("LSE_ONESTAGE_MAX_PARTS", "0")
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    for r in single:
        r.advance(60)
    monkeypatch.setenv("LSE_FUSED_BATCH", "1")
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(len(imgs))]
    tb = TileBatch(batch)
    for n in (1, 9, 50):
        tb.advance(n)
    check_same(batch, single)


def test_fused_batch_degenerate_and_forced_redo(monkeypatch):
    """Opt-in batched speculative pass with a zero-capacity fix list (every
    region tile redone) and a constant (degenerate) tile."""
    imgs = [tile(0), np.full((100, 80), 0.5), tile(2)]
    seeds = [L.SeedSpec(polygons=(square(6, 8, 70, 90),), inside_sign=-1)] * 3
    prm = [params("region", max_iters=40)] * 3
    monkeypatch.setenv("LSE_FINE_MAX_PX", "0")
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(3)]
    for r in single:
        r.advance(40)
    monkeypatch.setenv("LSE_FUSED_BATCH", "1")
    monkeypatch.setenv("LSE_FIX_CAP", "0")
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(3)]
    TileBatch(batch).advance(40)
    check_same(batch, single)
    assert batch[1].state.degenerate


def test_chunked_batch_advance_and_degenerate_tile():
    imgs = [tile(0), np.full((100, 80), 0.5), tile(2)]          # tile 1: constant image
    seeds = [L.SeedSpec(polygons=(square(6, 8, 70, 90),), inside_sign=-1)] * 3
    prm = [params("region", max_iters=40)] * 3
    single = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(3)]
    for r in single:
        r.advance(40)
    batch = [L.EvolutionRun(imgs[k], seeds[k], prm[k]) for k in range(3)]
    tb = TileBatch(batch)
    for n in (1, 7, 32):
        tb.advance(n)
    check_same(batch, single)
    assert batch[1].state.degenerate


def test_rgb8_tiles_decode_to_reference_luma():
    g = load_golden("luma")
    rgb = np.ascontiguousarray(np.tile(g["rgb"], (4, 3, 1)))     # 64 x 57 x 3
    luma = scenes.luma(rgb)
    assert np.array_equal(luma[:16, :19], g["luma"])
    seeds = L.SeedSpec(polygons=(square(5, 5, 50, 55),), inside_sign=1)
    for model in ("region", "edge"):
        prm = params(model, max_iters=25)
        a = _tile_run(rgb, seeds, prm)
        b = L.EvolutionRun(luma, seeds, prm)
        a.advance(25)
        b.advance(25)
        assert np.array_equal(a.state.phi, b.state.phi)


def test_c4_tiles_batch_matches_oracle_and_single_runs():
    n, size, iters = 4, 256, 30
    sc = [scenes.config4_tile(k, size, iters) for k in range(n)]
    seeds = [L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign) for s in sc]
    prm = [params(s.model, **s.params) for s in sc]
    res = run_tiles([s.image for s in sc], seeds, prm)
    for k, s in enumerate(sc):
        single = _tile_run(s.image, seeds[k], prm[k])
        single.advance(iters)
        assert np.array_equal(res[k].mask, single.mask())
        assert res[k].iterations == iters
    # tile 0 (region) and tile 1 (edge) against the oracle on the reference luma
    for k in (0, 1):
        p = prm[k]
        op = O.OracleParams(model=p.model.value, dt=p.dt, sigma2=p.sigma2, ts_reg=p.ts_reg,
                            max_iters=iters, conv_check_every=iters + 1,
                            sigma1=p.model_params.sigma1, ts_pre=p.model_params.ts_pre,
                            edge_gain=p.model_params.edge_gain)
        phi0 = O.rasterize_seeds(list(sc[k].polygons), sc[k].inside_sign, size, size)
        r = O.run_fixed(scenes.luma(sc[k].image), phi0, op, iters)
        mask = (r.phi > 0) if sc[k].inside_sign > 0 else (r.phi <= 0)
        assert np.array_equal(res[k].mask, mask)


def test_batch_rejects_mismatched_tiles():
    a = L.EvolutionRun(tile(0), L.SeedSpec(polygons=(square(6, 8, 70, 90),)), params("region"))
    b = L.EvolutionRun(tile(1, 96), L.SeedSpec(polygons=(square(6, 8, 70, 90),)),
                       params("region"))
    with pytest.raises(RuntimeError):
        TileBatch([a, b])


def test_sharded_runner_single_rank_equals_run_tiles():
    n, size, iters = 3, 128, 20
    sc = [scenes.config4_tile(k, size, iters) for k in range(n)]

    def make(k):
        s = sc[k]
        return s.image, L.SeedSpec(polygons=s.polygons, inside_sign=s.inside_sign), \
            params(s.model, **s.params)

    a = run_tiles_sharded(make, n, rank=0, world=1)
    b = run_tiles([make(k)[0] for k in range(n)], [make(k)[1] for k in range(n)],
                  [make(k)[2] for k in range(n)])
    for x, y in zip(a, b):
        assert np.array_equal(x.mask, y.mask) and x.iterations == y.iterations == iters
