"""GPU parity: the CUDA path through the drop-in API against the reference's
own outputs (golden fixtures made by tests/golden/make_golden.py) and the
oracle.  Bar: bit-exact phi wherever the reference's arithmetic is fully
reproducible (every edge-model run, every binary-state region run); for
region runs that carry a continuous field (reinit_period/reg_period != 1)
phi depends on c+/c-, whose last bits follow numpy's pairwise summation
order, so there the tolerance is 1e-12 relative to the phi range (far inside
the north star's 1e-4) and the zero-level masks must be identical."""
import hashlib
import warnings

import numpy as np
import pytest

import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import scenes
from conftest import load_golden

import lse_oracle as O

pytestmark = pytest.mark.gpu

TRAJ = ["traj_region_small", "traj_edge_small", "traj_region_field", "traj_region_mixed",
        "traj_edge_mixed", "traj_degenerate", "traj_odd_ts3", "traj_odd_ts5", "traj_odd_ts7",
        "traj_odd_edge_ts3", "traj_odd_edge_ts5", "traj_odd_edge_ts7", "traj_thin",
        "traj_a1", "traj_a1_cw2", "traj_a1_cw1", "traj_a1_edge", "traj_a2_edge",
        "traj_a5_region", "traj_a5_edge", "traj_instability", "traj_zhang_small",
        "traj_zhang_nu", "traj_a4_neg", "traj_a4_pos"]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def params_from(g):
    p = g["params"]
    model = L.ModelKind.from_name(str(g["model"]))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return L.default_params(model, dt=float(p[0]), sigma2=float(p[1]), ts_reg=int(p[2]),
                                reinit_period=int(p[3]), reg_period=int(p[4]),
                                max_iters=int(p[5]), conv_check_every=int(p[6]),
                                conv_window=int(p[7]), sigma1=float(p[8]), ts_pre=int(p[9]),
                                edge_gain=float(p[10]),
                                nu=float(g["nu"]) if "nu" in g else 1.0)


def exact_expected(prm):
    return prm.model is L.ModelKind.EDGE or (prm.reinit_period == 1 and prm.reg_period == 1)


def check_phi(got, want, exact):
    if exact:
        assert np.array_equal(got, want), f"max |dphi| = {np.abs(got - want).max():.3e}"
    else:
        rng = float(want.max() - want.min()) or 1.0
        assert np.abs(got - want).max() <= 1e-12 * rng
        assert np.array_equal(got > 0, want > 0)


@pytest.mark.parametrize("name", TRAJ)
def test_trajectory_matches_reference(name):
    g = load_golden(name)
    prm = params_from(g)
    seeds = L.SeedSpec(polygons=tuple(q for q in g["poly"]), inside_sign=int(g["inside_sign"]))
    r = L.EvolutionRun(g["image"], seeds, prm)
    err = -1
    try:
        for it in g["iters_recorded"]:
            r.advance(int(it) - r.state.iteration)
            phi = r.state.phi
            if f"phi_{it}" in g:
                check_phi(phi, g[f"phi_{it}"], exact_expected(prm))
            else:
                assert sha(phi) == str(g[f"sha_{it}"]), f"phi differs at iteration {it}"
                assert np.array_equal(np.packbits(phi > 0), g[f"mask_{it}"])
            if r.converged:
                break
        if int(g["instability_iteration"]) > 0:
            r.advance(prm.max_iters)
    except L.NumericalInstabilityError as e:
        err = e.iteration
    st = r.state
    assert err == int(g["instability_iteration"])
    assert st.iteration == int(g["final_iteration"])
    assert st.converged == bool(g["converged"])
    assert st.degenerate == bool(g["degenerate"])


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_north_star_configs_bit_exact(cfg):
    """C1 (256^2 region, dt=100, 5x5, 200 its) and C2 (1024^2 edge, 500 its):
    final phi identical to the reference's (SHA-256 of the float64 bytes)."""
    g = load_golden(f"traj_{cfg}")
    sc = scenes.config1() if cfg == "C1" else scenes.config2()
    prm = params_from(g)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    r = L.EvolutionRun(sc.image, seeds, prm)
    r.advance(sc.iters)
    st = r.state
    assert st.iteration == int(g["final_iteration"]) == sc.iters
    phi = st.phi
    assert np.array_equal(np.packbits(phi > 0), g[f"mask_{sc.iters}"])
    assert sha(phi) == str(g[f"sha_{sc.iters}"])
    fast, generic = r.path_counts()
    assert fast == sc.iters and generic == 0


def test_step_matches_reference():
    g = load_golden("step_edge")
    st = L.EvolutionState(phi=g["phi0"])
    prm = L.default_params(L.ModelKind.EDGE, sigma1=1.0, ts_pre=9)
    for k in range(3):
        st = L.step(st, g["image"], prm)
        assert st.iteration == k + 1
        assert np.array_equal(st.phi, g[f"phi_{k + 1}"])


def test_public_kernels_bit_exact():
    g = load_golden("kernels")
    for k, (s, ts) in enumerate(g["specs"]):
        out = L.convolve_same(g[f"conv_in_{k}"], L.gaussian_kernel(float(s), int(ts)))
        assert np.array_equal(out, g[f"conv_out_{k}"])
    fx, fy = L.gradient_central(g["grad_in"])
    assert np.array_equal(fx, g["grad_fx"]) and np.array_equal(fy, g["grad_fy"])
    assert np.array_equal(L.gradient_magnitude(g["grad_in"]), np.hypot(g["grad_fx"], g["grad_fy"]))
    for k in range(3):
        s1, ts, gain = g[f"edge_par_{k}"]
        assert np.array_equal(L.edge_function(g[f"edge_in_{k}"], float(s1), int(ts), float(gain)),
                              g[f"edge_out_{k}"])
    cp, cm = L.region_means(g["rm_img"], g["rm_phi"])
    assert abs(cp - g["rm_means"][0]) <= 1e-15 and abs(cm - g["rm_means"][1]) <= 1e-15
    seeds = L.SeedSpec(polygons=(g["rast_t1"], g["rast_t2"]), inside_sign=-1)
    assert np.array_equal(L.rasterize_seeds(seeds, 24, 24), g["rast_out"])
    seeds = L.SeedSpec(polygons=(g["rast_b1_poly"],), inside_sign=1)
    assert np.array_equal(L.rasterize_seeds(seeds, 128, 128), g["rast_b1_out"])


def test_velocities_match_oracle():
    rng = np.random.default_rng(5)
    img = rng.random((40, 52))
    phi = O.binarize(rng.standard_normal((40, 52)))
    phi = O.convolve_same(phi, O.gaussian_weights(1.0, 9))
    v, deg = L.region_velocity(img, phi)
    vo, dego = O.region_velocity(img, phi)
    assert deg == dego
    assert np.abs(v - vo).max() <= 1e-15
    gg = O.edge_function(img, 1.0, 9)
    assert np.array_equal(L.edge_velocity(gg, phi), O.edge_velocity(gg, phi))
    v, deg = L.region_velocity(np.full((12, 12), 0.5), np.where(rng.random((12, 12)) > .5, 1., -1.))
    assert deg and not v.any()


def test_zhang_velocity_matches_reference():
    g = load_golden("zhang")
    for k in range(4):
        v, deg = L.zhang_velocity(g[f"img_{k}"], g[f"phi_{k}"], float(g[f"nu_{k}"]))
        assert deg == bool(g[f"deg_{k}"])
        # c+/c- are correctly rounded on the device, numpy's pairwise mean can be
        # an ulp off: a few ulp of |v| (same bar as region_velocity below)
        want = g[f"v_{k}"]
        assert np.abs(v - want).max() <= 4 * np.finfo(float).eps * np.abs(want).max(), k
    v, deg = L.zhang_velocity(g["img_c"], g["phi_c"], 1.0)
    assert deg and not v.any()


@pytest.mark.parametrize("size,iters", [(512, 120), (1024, 40)])
def test_c5_density_crop_matches_oracle(size, iters):
    """C5's scene statistics at crop size: GPU phi == oracle phi after N its."""
    sc = scenes.config5_crop(size, iters)
    prm = L.default_params(L.ModelKind.REGION, **sc.params)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    r = L.EvolutionRun(sc.image, seeds, prm)
    r.advance(iters)
    phi = r.state.phi
    img64 = sc.image.astype(np.float64)
    phi0 = O.rasterize_seeds(sc.polygons, sc.inside_sign, size, size)
    ref = O.run_fixed(img64, phi0, O.OracleParams(model="region", dt=15.0, sigma2=1.5, ts_reg=9,
                                                  max_iters=iters, conv_check_every=iters + 1),
                      iters)
    assert ref.iteration == iters
    assert np.array_equal(phi, ref.phi)


@pytest.mark.parametrize("model", ["region", "edge"])
def test_uniform_skip_is_bit_identical_to_dense(model):
    """The exact uniform-window skip must not change a single bit."""
    sc = scenes.config5_crop(1024, 60)
    kw = dict(sc.params)
    if model == "edge":
        kw.update(sigma1=1.0, ts_pre=9)
    prm = L.default_params(L.ModelKind.from_name(model), **kw)
    seeds = L.SeedSpec(polygons=sc.polygons, inside_sign=sc.inside_sign)
    out = []
    for skip in (0, 1):
        r = L.EvolutionRun(sc.image, seeds, prm)
        r.set_native_option("skip_uniform", skip)
        r.advance(60)
        out.append(r.state.phi)
    assert np.array_equal(out[0], out[1])
