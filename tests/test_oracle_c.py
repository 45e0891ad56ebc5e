"""The C restatement (CPU baseline) is pinned bit-exact to the reference's
golden outputs, like the numpy oracle."""
import hashlib

import numpy as np
import pytest

import lse_oracle as O
import lse_oracle_c as OC
from conftest import load_golden
from test_oracle_golden import _params, _phi0


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["traj_region_small", "traj_edge_small", "traj_region_field",
                                  "traj_region_mixed", "traj_edge_mixed", "traj_degenerate",
                                  "traj_odd_ts3", "traj_odd_edge_ts7", "traj_thin", "traj_a1",
                                  "traj_a1_cw2", "traj_a1_cw1", "traj_a2_edge",
                                  "traj_a5_region", "traj_instability", "traj_C1",
                                  "traj_zhang_small", "traj_zhang_nu", "traj_a4_neg",
                                  "traj_a4_pos"])
def test_c_oracle_matches_reference(name):
    g = load_golden(name)
    if name == "traj_C1":
        from paper_1409_7474_b200 import scenes
        sc = scenes.config1()
        img = sc.image.astype(np.float64)
        phi0 = O.rasterize_seeds(list(sc.polygons), sc.inside_sign, 256, 256)
    else:
        img = g["image"]
        phi0 = _phi0(g, img.shape)
    p = _params(g)
    r = OC.COracleRun(img, phi0, p, O.gaussian_weights)
    err = 0
    for it in g["iters_recorded"]:
        err = r.advance(int(it) - r.iteration)
        if err:
            break
        if f"phi_{it}" in g:
            assert np.array_equal(r.phi, g[f"phi_{it}"])
        else:
            assert sha(r.phi) == str(g[f"sha_{it}"])
        if r.converged:
            break
    if int(g["instability_iteration"]) > 0 and not err:
        err = r.advance(p.max_iters)
    assert err == max(0, int(g["instability_iteration"]))
    assert r.iteration == int(g["final_iteration"])
    assert r.converged == bool(g["converged"])
    assert r.degenerate == bool(g["degenerate"])


def test_c_edge_function_bit_exact():
    g = load_golden("kernels")
    lib = OC.load()
    for k in range(3):
        s1, ts, gain = g[f"edge_par_{k}"]
        img = np.ascontiguousarray(g[f"edge_in_{k}"])
        w = np.ascontiguousarray(O.gaussian_weights(float(s1), int(ts)))
        out = np.empty_like(img)
        lib.oracle_edge_function(img.ctypes.data_as(OC._dp), img.shape[0], img.shape[1],
                                 w.ctypes.data_as(OC._dp), int(ts), float(gain),
                                 out.ctypes.data_as(OC._dp))
        assert np.array_equal(out, g[f"edge_out_{k}"])


def _band_scene(k, h=72, w=64, seed=9):
    rng = np.random.default_rng(seed)
    base = np.array([0.25, 0.30, 0.28, 0.45])[:k]
    fg = np.array([0.60, 0.62, 0.65, 0.35])[:k]
    bands = base[:, None, None] + 0.05 * rng.standard_normal((k, h, w))
    bands[:, 20:55, 15:50] = fg[:, None, None] + 0.04 * rng.standard_normal((k, 35, 35))
    return np.clip(bands, 0, 1)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_c_oracle_bands_match_numpy_restatement(k):
    """The C restatement of C3's multi-band term equals the numpy one bit for
    bit (and K = 1 is the region model: pinned to the reference goldens)."""
    bands = _band_scene(k)
    h, w = bands.shape[1:]
    phi0 = O.rasterize_seeds([np.array([[4., 4.], [60., 4.], [60., 68.], [4., 68.]])], -1, w, h)
    p = O.OracleParams(model="region", dt=15.0, sigma2=1.0, ts_reg=9, max_iters=60,
                       conv_check_every=61)
    ref = O.run_fixed(bands if k > 1 else bands[0], phi0, p, 60)
    r = OC.COracleRun(bands, phi0, p, O.gaussian_weights)
    r.advance(60)
    assert r.iteration == 60
    assert np.array_equal(r.phi, ref.phi)
    if k == 1:
        r1 = OC.COracleRun(bands[0], phi0, p, O.gaussian_weights)
        r1.advance(60)
        assert np.array_equal(r1.phi, r.phi)


def test_c_oracle_thread_count_does_not_change_results():
    bands = _band_scene(2, seed=3)
    phi0 = O.rasterize_seeds([np.array([[4., 4.], [60., 4.], [60., 68.], [4., 68.]])], 1, 64, 72)
    p = O.OracleParams(model="region", dt=15.0, sigma2=1.0, ts_reg=9, max_iters=30,
                       conv_check_every=31)
    out = []
    for n in (1, 4):
        OC.set_threads(n)
        r = OC.COracleRun(bands, phi0, p, O.gaussian_weights)
        r.advance(30)
        out.append(r.phi.copy())
    OC.set_threads(0)
    assert np.array_equal(out[0], out[1])
