"""The reference's own behavioural tests (pkg/tests/test_engine.py, test_models,
test_grid, acceptance A1/A3/A5/A6/A9/A10), re-run through the drop-in API on
the device."""
import warnings

import numpy as np
import pytest

import paper_1409_7474_b200 as L
from conftest import dice, square, two_region

pytestmark = pytest.mark.gpu

A1_SEED = L.SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1)


def edge_params(**kw):
    kw.setdefault("max_iters", 300)
    return L.default_params(L.ModelKind.EDGE, dt=15.0, sigma2=1.0, ts_reg=9, sigma1=1.0,
                            ts_pre=9, **kw)


def test_a1_region_reproduction():
    image, truth = two_region()
    res = L.run(image, A1_SEED, L.default_params(L.ModelKind.REGION, max_iters=300))
    assert res.converged and res.iterations == 40
    assert dice(res.mask, truth) >= 0.99
    assert res.object_sign == -1 and res.wall_time > 0


def test_a2_edge_position_sensitivity():
    image, truth = two_region(256, 48, 208, 0.41, 0.59)
    out = L.run(image, L.SeedSpec(polygons=(square(36, 36, 220, 220),)), edge_params())
    assert dice(out.mask, truth) >= 0.98
    cross = L.run(image, L.SeedSpec(polygons=(square(20, 20, 120, 120),)), edge_params())
    assert (not cross.mask.any()) or dice(cross.mask, truth) < 0.5


def test_a3_sign_robustness():
    image, truth = two_region()
    d = {}
    for sign in (-1, 1):
        seed = L.SeedSpec(polygons=(square(28, 28, 100, 100),), inside_sign=sign)
        d["r", sign] = dice(L.run(image, seed, L.default_params(L.ModelKind.REGION)).mask, truth)
        d["e", sign] = dice(L.run(image, seed, edge_params()).mask, truth)
    assert d["r", -1] >= 0.99 and d["r", 1] >= 0.99
    assert d["e", -1] >= 0.8 and d["e", 1] < 0.5


def test_a4_zhang_sign_sensitivity():
    """test_acceptance.py:95-105: the mean-separation baseline depends on the sign."""
    image, truth = two_region()
    ds = {}
    for sign in (-1, 1):
        seed = L.SeedSpec(polygons=(square(28, 28, 100, 100),), inside_sign=sign)
        r = L.run(image, seed, L.default_params(L.ModelKind.ZHANG, nu=1.0, max_iters=1000))
        ds[sign] = dice(r.mask, truth)
    assert ds[-1] >= 0.95 and ds[1] < 0.5


def test_zhang_init_state_is_binary():
    image, _ = two_region()
    st = L.init_state(image, A1_SEED, L.default_params(L.ModelKind.ZHANG))
    assert set(np.unique(st.phi)) == {-1.0, 1.0} and st.iteration == 0


def test_a5_noise_robustness():
    image, truth = two_region()
    rd, ed = [], []
    for s in range(5):
        noisy = np.clip(image + np.random.default_rng(s).normal(0.0, 0.2, image.shape), 0, 1)
        rd.append(dice(L.run(noisy, A1_SEED, L.default_params(L.ModelKind.REGION)).mask, truth))
        ed.append(dice(L.run(noisy, L.SeedSpec(polygons=(square(20, 20, 108, 108),)),
                             edge_params()).mask, truth))
    assert min(rd) >= 0.95 and max(ed) < 0.9


def test_a6_affine_invariance_every_checkpoint():
    image, _ = two_region()
    p = L.default_params(L.ModelKind.REGION)
    r1 = L.EvolutionRun(image, A1_SEED, p)
    r2 = L.EvolutionRun(0.5 * image + 0.1, A1_SEED, p)
    while True:
        r1.advance(p.conv_check_every)
        r2.advance(p.conv_check_every)
        assert np.array_equal(r1.mask(), r2.mask())
        if (r1.converged and r2.converged) or r1.state.iteration >= p.max_iters:
            break
    assert r1.converged and r2.converged and r1.state.iteration == r2.state.iteration


def test_a9_determinism_and_mirror():
    image, _ = two_region()
    p = L.default_params(L.ModelKind.REGION)
    a, b = L.run(image, A1_SEED, p), L.run(image, A1_SEED, p)
    assert np.array_equal(a.mask, b.mask) and a.iterations == b.iterations
    poly = A1_SEED.polygons[0].copy()
    poly[:, 0] = image.shape[1] - poly[:, 0]
    m = L.run(image[:, ::-1], L.SeedSpec(polygons=(poly,), inside_sign=-1), p)
    assert np.array_equal(m.mask, a.mask[:, ::-1]) and m.iterations == a.iterations


def test_a9_edge_interior_never_grows():
    image, _ = two_region(256, 48, 208, 0.41, 0.59)
    ep = edge_params()
    st = L.init_state(image, L.SeedSpec(polygons=(square(36, 36, 220, 220),)), ep)
    counts = []
    for _ in range(20):
        st = L.step(st, image, ep)
        counts.append(int((L.binarize(st.phi) <= 0).sum()))
    assert all(b <= a for a, b in zip(counts, counts[1:]))


def test_a10_dt40_warns_and_stays_finite():
    image, truth = two_region()
    with pytest.warns(RuntimeWarning, match="unstable"):
        p = L.default_params(L.ModelKind.REGION, dt=40.0)
    r = L.EvolutionRun(image, A1_SEED, p)
    while not r.converged and r.state.iteration < p.max_iters:
        r.advance(p.conv_check_every)
        assert np.isfinite(r.state.phi).all()
    assert dice(r.mask(), truth) >= 0.99


def test_instability_names_iteration_and_keeps_last_state():
    image, _ = two_region()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        p = L.default_params(L.ModelKind.REGION, dt=1e308, reinit_period=0)
    r = L.EvolutionRun(image, A1_SEED, p)
    with pytest.raises(L.NumericalInstabilityError) as e:
        r.advance(10)
    assert e.value.iteration == 1 and "instability" in str(e.value)
    assert r.state.iteration == 0
    assert set(np.unique(r.state.phi)) == {-1.0, 1.0}
    st = L.init_state(image, A1_SEED, p)
    with pytest.raises(L.NumericalInstabilityError):
        L.step(st, image, p)


def test_degenerate_fixed_point():
    image = np.full((32, 32), 0.5)
    seeds = L.SeedSpec(polygons=(square(0, 0, 32, 16),), inside_sign=-1)
    p = L.default_params(L.ModelKind.REGION)
    st = L.init_state(image, seeds, p)
    before = L.binarize(st.phi)
    st = L.step(st, image, p)
    assert st.degenerate and np.array_equal(L.binarize(st.phi), before)


def test_resumable_advance_matches_single_run():
    image, _ = two_region()
    p = L.default_params(L.ModelKind.REGION)
    whole = L.run(image, A1_SEED, p)
    r = L.EvolutionRun(image, A1_SEED, p)
    while not r.converged and r.state.iteration < p.max_iters:
        r.advance(7)
    assert r.state.iteration == whole.iterations
    assert np.array_equal(r.mask(), whole.mask)


def test_max_iters_one_and_advance_zero():
    image, _ = two_region()
    res = L.run(image, A1_SEED, L.default_params(L.ModelKind.REGION, max_iters=1))
    assert res.iterations == 1 and not res.converged
    r = L.EvolutionRun(image, A1_SEED, L.default_params(L.ModelKind.REGION))
    assert r.advance(0).iteration == 0


def test_step_after_convergence_rejected():
    image, _ = two_region()
    r = L.EvolutionRun(image, A1_SEED, L.default_params(L.ModelKind.REGION))
    r.advance(1000)
    assert r.converged
    with pytest.raises(ValueError):
        L.step(r.state, image, r.params)


def test_state_snapshot_is_immutable_and_reinjectable():
    image, _ = two_region()
    p = L.default_params(L.ModelKind.REGION)
    r = L.EvolutionRun(image, A1_SEED, p)
    r.advance(5)
    snap = r.state          # phi not read yet
    r.advance(5)
    phi5 = snap.phi         # must still be the iteration-5 field
    ref = L.EvolutionRun(image, A1_SEED, p)
    ref.advance(5)
    assert np.array_equal(phi5, ref.state.phi)
    r.state = L.EvolutionState(phi=phi5, iteration=5)   # re-inject (G*b form -> bit path)
    r.advance(5)
    ref.advance(5)
    assert np.array_equal(r.state.phi, ref.state.phi)
    assert r.path_counts()[1] <= 1   # one exact fp64 iteration re-derives the bit state


def test_grid_and_model_unit_behaviour():
    assert np.array_equal(L.binarize(np.array([[0.3, -0.2, 0.0]])), np.array([[1.0, -1.0, -1.0]]))
    assert L.region_means(np.array([[0.1, 0.9]]), np.array([[0.0, -1.0]])) == (0.1, 0.9)
    with pytest.raises(L.DegeneratePartitionError):
        L.region_means(np.random.default_rng(1).random((4, 4)), np.ones((4, 4)))
    with pytest.raises(L.DegenerateSeedError):
        L.rasterize_seeds(L.SeedSpec(polygons=(square(100, 100, 120, 120),)), 8, 8)
    with pytest.raises(L.DegenerateSeedError):
        L.rasterize_seeds(L.SeedSpec(polygons=(square(-5, -5, 50, 50),)), 8, 8)
    phi = np.tile(np.arange(32.0) - 15.5, (32, 1))
    v, deg = L.region_velocity(np.random.default_rng(4).random((32, 32)), phi)
    assert not deg and abs(np.abs(v).max() - 1.0) <= 1e-12
    g = L.edge_function(np.full((16, 16), 0.4), 1.0, 9)
    assert np.allclose(g[5:-5, 5:-5], 1.0, atol=1e-12) and (g > 0).all() and (g <= 1).all()


def test_plain_c_caller_matches_python_api(tmp_path):
    """examples/c_abi_region.c drives the C ABI directly (no Python in the loop)
    and must reach the same result as lse.run through the Python API."""
    import hashlib
    import os
    import subprocess
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "c_abi_region"
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(repo, "include"),
                           os.path.join(repo, "examples", "c_abi_region.c"),
                           "-L", os.path.join(repo, "paper_1409_7474_b200", "_lib"), "-llse_b200",
                           "-lm", "-o", str(exe)])
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(repo, "paper_1409_7474_b200", "_lib"))
    it, conv, hsh = subprocess.check_output([str(exe)], env=env).decode().split()
    image = np.full((128, 128), 0.8)
    image[40:88, 40:88] = 0.2
    res = L.run(image, A1_SEED, L.default_params(L.ModelKind.REGION, max_iters=300))
    h = 1469598103934665603
    for q in res.mask.astype(np.uint8).ravel():
        h = ((h ^ int(q)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    assert int(it) == res.iterations and bool(int(conv)) == res.converged
    assert int(hsh, 16) == h


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_image_rejected(dtype, bad):
    """as_field's ValueError (grid.py:24-31); float32 region images are checked
    by the device's image statistics pass instead of a host scan."""
    img = np.full((70, 90), 0.4, dtype=dtype)
    img[33, 57] = bad
    seeds = L.SeedSpec(polygons=(square(5, 5, 60, 50),), inside_sign=-1)
    for kind in (L.ModelKind.REGION, L.ModelKind.EDGE):
        with pytest.raises(ValueError, match="non-finite"):
            L.EvolutionRun(img, seeds, L.default_params(kind))
