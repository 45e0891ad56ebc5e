"""The oracle is pinned against the reference's own outputs (bit-exact)."""
import hashlib

import numpy as np
import pytest

import lse_oracle as O
from conftest import load_golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_gaussian_and_convolution_bit_exact():
    g = load_golden("kernels")
    for k, (s, ts) in enumerate(g["specs"]):
        w = O.gaussian_weights(float(s), int(ts))
        assert np.array_equal(w, g[f"w_{k}"])
        assert np.array_equal(O.convolve_same(g[f"conv_in_{k}"], w), g[f"conv_out_{k}"])


def test_gradient_and_edge_function_bit_exact():
    g = load_golden("kernels")
    fx, fy = O.gradient_central(g["grad_in"])
    assert np.array_equal(fx, g["grad_fx"]) and np.array_equal(fy, g["grad_fy"])
    for k in range(3):
        s1, ts, gain = g[f"edge_par_{k}"]
        out = O.edge_function(g[f"edge_in_{k}"], float(s1), int(ts), float(gain))
        assert np.array_equal(out, g[f"edge_out_{k}"])


def test_region_means_and_pairwise_restatement():
    g = load_golden("kernels")
    assert np.array_equal(np.array(O.region_means(g["rm_img"], g["rm_phi"])), g["rm_means"])
    img, phi = g["rm_img"], g["rm_phi"]
    pos = phi >= 0
    assert O.pairwise_sum(img[pos]) / pos.sum() == g["rm_means"][0]


def test_rasterize_bit_exact():
    g = load_golden("kernels")
    out = O.rasterize_seeds([g["rast_t1"], g["rast_t2"]], -1, 24, 24)
    assert np.array_equal(out, g["rast_out"])
    out = O.rasterize_seeds([g["rast_b1_poly"]], 1, 128, 128)
    assert np.array_equal(out, g["rast_b1_out"])


def test_zhang_velocity_bit_exact():
    g = load_golden("zhang")
    for k in range(4):
        v, deg = O.zhang_velocity(g[f"img_{k}"], g[f"phi_{k}"], float(g[f"nu_{k}"]))
        assert np.array_equal(v, g[f"v_{k}"]) and deg == bool(g[f"deg_{k}"])
    v, deg = O.zhang_velocity(g["img_c"], g["phi_c"], 1.0)
    assert deg and bool(g["deg_c"]) and not v.any() and not g["v_c"].any()


def test_glibc_hypot_restatement():
    rng = np.random.default_rng(0)
    for e in (-200, -20, 0, 20, 200):
        x = rng.standard_normal(300) * 10.0 ** e
        y = rng.standard_normal(300) * 10.0 ** (e - 3)
        assert all(O.glibc_hypot(a, b) == np.hypot(a, b) for a, b in zip(x, y))


def _params(g):
    p = g["params"]
    return O.OracleParams(model=str(g["model"]), dt=float(p[0]), sigma2=float(p[1]),
                          ts_reg=int(p[2]), reinit_period=int(p[3]), reg_period=int(p[4]),
                          max_iters=int(p[5]), conv_check_every=int(p[6]),
                          conv_window=int(p[7]), sigma1=float(p[8]), ts_pre=int(p[9]),
                          edge_gain=float(p[10]),
                          nu=float(g["nu"]) if "nu" in g else 1.0,
                          mu=float(g["mu"]) if "mu" in g else 0.1)


def _phi0(g, shape):
    polys = [q for q in g["poly"]]
    phi0 = O.rasterize_seeds(polys, int(g["inside_sign"]), shape[1], shape[0])
    if str(g["model"]) == "cv":                  # init_state: distance field (engine.py:129-132)
        phi0 = -O.signed_distance(phi0 > 0)
    return phi0


@pytest.mark.parametrize("name", ["traj_region_small", "traj_edge_small", "traj_region_field",
                                  "traj_region_mixed", "traj_edge_mixed", "traj_degenerate",
                                  "traj_odd_ts3", "traj_odd_ts5", "traj_odd_ts7",
                                  "traj_odd_edge_ts3", "traj_odd_edge_ts5", "traj_odd_edge_ts7",
                                  "traj_thin", "traj_a1", "traj_a1_cw2", "traj_a1_cw1",
                                  "traj_a1_edge", "traj_a2_edge", "traj_a5_region",
                                  "traj_a5_edge", "traj_instability", "traj_zhang_small",
                                  "traj_zhang_nu", "traj_a4_neg", "traj_a4_pos",
                                  "traj_cv_small", "traj_cv_a7"])
def test_oracle_trajectories_bit_exact(name):
    g = load_golden(name)
    img = g["image"]
    p = _params(g)
    r = O.OracleRun(img, _phi0(g, img.shape), p)
    err = -1
    try:
        for it in g["iters_recorded"]:
            r.advance(int(it) - r.iteration)
            if f"phi_{it}" in g:
                assert np.array_equal(r.phi, g[f"phi_{it}"]), f"phi differs at {it}"
            else:
                assert sha(r.phi) == str(g[f"sha_{it}"]), f"phi hash differs at {it}"
            if r.converged:
                break
        if int(g["instability_iteration"]) > 0:
            r.advance(p.max_iters)
    except O.OracleInstability as e:
        err = e.iteration
    assert err == int(g["instability_iteration"])
    assert r.iteration == int(g["final_iteration"])
    assert r.converged == bool(g["converged"])
    assert r.degenerate == bool(g["degenerate"])


def test_luma_restatement_matches_reference_loader():
    """scenes.luma (the C4 decode the device restates) == fileio._luma / 255."""
    from paper_1409_7474_b200 import scenes
    g = load_golden("luma")
    assert np.array_equal(scenes.luma(g["rgb"]), g["luma"])


def test_band_restatement_reduces_to_region_model():
    """C3's multi-band restatement with one band is region_velocity exactly, and
    runs the reference's region trajectory bit for bit (the pin for K > 1)."""
    rng = np.random.default_rng(9)
    img, phi = rng.random((21, 17)), rng.standard_normal((21, 17))
    v1, d1 = O.region_velocity(img, phi)
    vk, dk = O.region_velocity_bands(img[None], phi)
    assert d1 == dk and np.array_equal(v1, vk)
    g = load_golden("traj_region_small")
    img = g["image"]
    r = O.OracleRun(img[None], _phi0(g, img.shape), _params(g))
    for it in g["iters_recorded"]:
        r.advance(int(it) - r.iteration)
        assert np.array_equal(r.phi, g[f"phi_{it}"])


def test_cv_units_bit_exact():
    """signed_distance (exact EDT restatement), curvature, cv_velocity vs the reference."""
    g = load_golden("cv_units")
    for k in range(3):
        assert np.array_equal(O.signed_distance(g[f"mask_{k}"]), g[f"sd_{k}"])
        assert np.array_equal(O.curvature(g[f"f_{k}"]), g[f"curv_{k}"])
        assert np.array_equal(O.cv_velocity(g[f"img_{k}"], g[f"f_{k}"], 0.1 * (k + 1)), g[f"v_{k}"])
