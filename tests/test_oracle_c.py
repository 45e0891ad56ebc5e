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
