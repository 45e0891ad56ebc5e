"""Row-strip decomposition on the CPU: the strip driver and both
communicators (in-process, and torch.distributed over gloo with world_size 2)
drive the oracle-backed stand-in (tests/strip_mock.py); every strip layout
must reproduce the single-grid oracle trajectory."""
import os
import socket
import warnings

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lse_oracle as O
import paper_1409_7474_b200 as L
from paper_1409_7474_b200.strips import (LocalComm, DistComm, StripDriver, plan_strips,
                                         strip_rows, WORD_ROWS)
from conftest import square
from strip_mock import MockStrip


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def scene(h=150, w=70, seed=3):
    rng = np.random.default_rng(seed)
    img = np.full((h, w), 0.25)
    img[30:110, 20:55] = 0.7
    img = np.clip(img + 0.08 * rng.standard_normal((h, w)), 0, 1)
    seeds = L.SeedSpec(polygons=(square(8, 12, 60, 130),), inside_sign=-1)
    return img, seeds


def oracle_run(img, seeds, prm, iters):
    op = O.OracleParams(model=prm.model.value, dt=prm.dt, sigma2=prm.sigma2, ts_reg=prm.ts_reg,
                        max_iters=prm.max_iters, conv_check_every=prm.conv_check_every,
                        conv_window=prm.conv_window, sigma1=prm.model_params.sigma1,
                        ts_pre=prm.model_params.ts_pre, edge_gain=prm.model_params.edge_gain,
                        nu=prm.model_params.nu)
    phi0 = O.rasterize_seeds([np.asarray(q, float) for q in seeds.polygons], seeds.inside_sign,
                             img.shape[1], img.shape[0])
    r = O.OracleRun(img, phi0, op)
    r.advance(iters)
    return r


@pytest.mark.parametrize("h,world", [(150, 1), (150, 2), (150, 5), (64, 2), (33, 2), (1000, 7)])
def test_plan_strips_partition_word_rows(h, world):
    wins = plan_strips(h, 10, world)
    hr = (h + 31) // 32
    assert wins[0].wr0 == 0 and wins[-1].wr1 == hr
    for a, b in zip(wins, wins[1:]):
        assert a.wr1 == b.wr0
    for w in wins:
        assert w.y_lo % WORD_ROWS == 0 and w.own_lo in (0, 1)
        assert w.own_hi - w.own_lo == w.wr1 - w.wr0
        assert w.has_up == (w.wr0 > 0) and w.has_down == (w.wr1 < hr)
        lo, hi = w.own_rows
        assert w.y_lo <= lo < hi <= w.y_hi
        assert lo - w.y_lo == (WORD_ROWS if w.has_up else 0)
        assert w.y_hi - hi == (min(WORD_ROWS, h - hi) if w.has_down else 0)
    with pytest.raises(ValueError):
        plan_strips(h, 10, hr + 1)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("model,world,kw", [
    ("region", 2, {}), ("region", 4, {}), ("edge", 3, {}), ("zhang", 2, {}),
    ("region", 3, {"conv_check_every": 3, "conv_window": 2, "max_iters": 80}),
])
def test_local_strips_match_single_grid(model, world, kw, fused):
    """Both protocols of the driver: update -> halo -> partition -> allgather ->
    finalize, and the one-pass one (partition + next update -> allgather ->
    finalize (+ fix / redo) -> halo, the owed partition flushed at the end)."""
    img, seeds = scene()
    kw.setdefault("max_iters", 25)
    prm = params(model, **kw)
    iters = prm.max_iters
    ref = oracle_run(img, seeds, prm, iters)
    wins = plan_strips(img.shape[0], img.shape[1], world)
    strips = [MockStrip(strip_rows(img, w), w, seeds, prm) for w in wins]
    drv = StripDriver(strips, LocalComm(strips), fused=fused)
    assert drv.fused == fused
    drv.setup()
    st = drv.advance(iters)
    phi = np.concatenate([s.own_phi() for s in strips])
    assert np.array_equal(phi, ref.phi)
    assert all(s.iteration == ref.iteration for s in st)
    assert all(bool(s.converged) == ref.converged for s in st)


def test_degenerate_seed_is_global():
    img, _ = scene()
    seeds = L.SeedSpec(polygons=(square(0, 0, 70, 150),), inside_sign=1)   # covers everything
    wins = plan_strips(img.shape[0], img.shape[1], 2)
    prm = params("region")
    strips = [MockStrip(strip_rows(img, w), w, seeds, prm) for w in wins]
    with pytest.raises(L.DegenerateSeedError):
        StripDriver(strips, LocalComm(strips)).setup()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, model, iters, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img, seeds = scene()
        prm = params(model, max_iters=iters, conv_check_every=4, conv_window=2)
        win = plan_strips(img.shape[0], img.shape[1], world)[rank]
        strip = MockStrip(strip_rows(img, win), win, seeds, prm)
        drv = StripDriver([strip], DistComm(strip))
        drv.setup()
        st = drv.advance(iters)[0]
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), phi=strip.own_phi(),
                 it=st.iteration, conv=st.converged)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("model", ["region", "edge"])
def test_gloo_world2_matches_single_grid(model, tmp_path):
    world, iters = 2, 40
    mp.spawn(_gloo_worker, args=(world, _free_port(), model, iters, str(tmp_path)),
             nprocs=world, join=True)
    img, seeds = scene()
    ref = oracle_run(img, seeds, params(model, max_iters=iters, conv_check_every=4,
                                        conv_window=2), iters)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert np.array_equal(np.concatenate([o["phi"] for o in outs]), ref.phi)
    for o in outs:
        assert int(o["it"]) == ref.iteration and bool(o["conv"]) == ref.converged
