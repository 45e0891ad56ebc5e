"""Row strips on the device: G strips of one grid, driven on one
GPU exactly as G ranks would drive them (update -> halo exchange -> partition
-> partial allgather -> finalize), must reproduce the single-run trajectory
bit-for-bit."""
import warnings

import numpy as np
import pytest

import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from paper_1409_7474_b200.strips import run_local_strips
from conftest import square

pytestmark = pytest.mark.gpu


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return L.default_params(L.ModelKind.from_name(model), **kw)


def scene(h=150, w=70, seed=3):
    rng = np.random.default_rng(seed)
    img = np.full((h, w), 0.25)
    img[30:110, 20:55] = 0.7
    img = np.clip(img + 0.08 * rng.standard_normal((h, w)), 0, 1)
    return img, L.SeedSpec(polygons=(square(8, 12, 60, 130),), inside_sign=-1)


def single(img, seeds, prm, iters):
    r = L.EvolutionRun(img, seeds, prm)
    r.advance(iters)
    return r


def check(img, seeds, prm, iters, world):
    ref = single(img, seeds, prm, iters)
    _, strips, st = run_local_strips(img, seeds, prm, world, iters)
    phi = np.concatenate([s.own_phi() for s in strips])
    assert np.array_equal(phi, ref.state.phi), np.abs(phi - ref.state.phi).max()
    mask = np.concatenate([s.own_mask(seeds.inside_sign) for s in strips]).astype(bool)
    assert np.array_equal(mask, ref.mask())
    for s in st:
        assert s.iteration == ref.state.iteration and bool(s.converged) == ref.converged


@pytest.mark.parametrize("model,world", [("region", 2), ("region", 4), ("edge", 3),
                                         ("zhang", 2)])
def test_small_scene_strips(model, world):
    img, seeds = scene()
    check(img, seeds, params(model, max_iters=30), 30, world)


def test_strips_converge_together():
    img, seeds = scene()
    check(img, seeds, params("region", max_iters=300, conv_check_every=3, conv_window=2), 300, 3)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_c5_crop_strips(world):
    sc = scenes.config5_crop(1024, 60)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    check(sc.image, seeds, params("region", **sc.params), 60, world)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_c5_crop_strips_fused(world, monkeypatch):
    """Unsplit units (as at full size): every strip runs the one-pass
    iteration (lse_strip_fused: partition + speculative update -> partial
    exchange -> check / fix / redo -> halos) and reproduces the single run."""
    monkeypatch.setenv("LSE_SPLIT_PARTS", "1")
    sc = scenes.config5_crop(1024, 60)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    prm = params("region", **sc.params)
    ref = single(sc.image, seeds, prm, 60)
    drv, strips, st = run_local_strips(sc.image, seeds, prm, world, 60)
    assert drv.fused
    phi = np.concatenate([s.own_phi() for s in strips])
    assert np.array_equal(phi, ref.state.phi), np.abs(phi - ref.state.phi).max()
    for s in st:
        assert s.iteration == ref.state.iteration


def test_small_strips_fused_converge(monkeypatch):
    """Border-only strips on the one-pass iteration, converging mid-run."""
    monkeypatch.setenv("LSE_SPLIT_PARTS", "1")
    img, seeds = scene()
    prm = params("region", max_iters=300, conv_check_every=3, conv_window=2)
    ref = single(img, seeds, prm, 300)
    drv, strips, st = run_local_strips(img, seeds, prm, 3, 300)
    assert drv.fused
    phi = np.concatenate([s.own_phi() for s in strips])
    assert np.array_equal(phi, ref.state.phi)
    for s in st:
        assert s.iteration == ref.state.iteration and bool(s.converged) == ref.converged


def test_strip_degenerate_seed_is_global():
    img, _ = scene()
    seeds = L.SeedSpec(polygons=(square(0, 0, 70, 150),), inside_sign=1)
    with pytest.raises(L.DegenerateSeedError):
        run_local_strips(img, seeds, params("region"), 2, 1)


def test_nccl_communicator_world1():
    """The NCCL communicator path (allreduce of the image range, allgather of
    the partials on the strip's stream) in a one-rank process group."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_1409_7474_b200.strips import DeviceStrip, DistComm, StripDriver, plan_strips
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        img, seeds = scene()
        prm = params("region", max_iters=40)
        win = plan_strips(img.shape[0], img.shape[1], 1)[0]
        strip = DeviceStrip(img, win, seeds, prm)
        drv = StripDriver([strip], DistComm(strip))
        drv.setup()
        st = drv.advance(20)[0]
        strip.reset()                       # the bench's job: reset + initialize + advance
        drv.initialize()
        st = drv.advance(40)[0]
        ref = single(img, seeds, prm, 40)
        assert st.iteration == ref.state.iteration
        assert np.array_equal(strip.own_phi(), ref.state.phi)
    finally:
        dist.destroy_process_group()
