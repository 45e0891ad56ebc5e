"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array in the fixtures is produced by `lsekit` 0.1.0 itself
(/root/reference/pkg/src/lsekit); the repo's oracle and the CUDA path are
then checked against these files.  Large states are pinned by SHA-256 of
the float64 phi bytes plus the packed final mask.  Nothing here is used at
run time on the GPU box except the committed .npz outputs.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import lsekit  # noqa: E402  (the reference)
from lsekit import (EvolutionRun, EvolutionState, ModelKind, SeedSpec,  # noqa: E402
                    NumericalInstabilityError, binarize, convolve_same,
                    default_params, edge_function, gaussian_kernel,
                    gradient_central, rasterize_seeds, region_means, step,
                    zhang_velocity)

import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "lse_scenes", os.path.join(REPO, "paper_1409_7474_b200", "scenes.py"))
scenes = importlib.util.module_from_spec(_spec)   # seeded inputs only
sys.modules["lse_scenes"] = scenes
_spec.loader.exec_module(scenes)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def square(x0, y0, x1, y1):
    return np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], dtype=float)


def two_region(size=128, obj0=40, obj1=88, io=0.2, ib=0.8):
    img = np.full((size, size), ib)
    img[obj0:obj1, obj0:obj1] = io
    return img


def params(model, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        return default_params(model, **kw)


def kernels_fixture():
    rng = np.random.default_rng(7)
    out = {}
    specs = [(1.0, 9), (1.5, 9), (1.0, 5), (2.0, 7), (1.3, 7), (0.7, 3), (1.0, 1), (3.0, 15)]
    for k, (s, ts) in enumerate(specs):
        w = gaussian_kernel(s, ts).axis_weights
        f = rng.standard_normal((13 + k, 17 + 2 * k))
        out[f"w_{k}"] = w
        out[f"conv_in_{k}"] = f
        out[f"conv_out_{k}"] = convolve_same(f, gaussian_kernel(s, ts))
    out["specs"] = np.array(specs)
    f = rng.standard_normal((11, 9)) * 3
    fx, fy = gradient_central(f)
    out["grad_in"], out["grad_fx"], out["grad_fy"] = f, fx, fy
    for k, (s1, ts, gain) in enumerate([(1.0, 9, 255.0), (1.5, 9, 255.0), (1.0, 5, 1.0)]):
        img = rng.random((24 + k, 31 - k))
        out[f"edge_in_{k}"] = img
        out[f"edge_out_{k}"] = edge_function(img, s1, ts, gain)
        out[f"edge_par_{k}"] = np.array([s1, ts, gain])
    img, phi = rng.random((16, 16)), rng.standard_normal((16, 16))
    out["rm_img"], out["rm_phi"] = img, phi
    out["rm_means"] = np.array(region_means(img, phi))
    t1 = np.array([[1.0, 1.0], [9.0, 2.0], [3.0, 8.0]])
    t2 = np.array([[12.0, 10.0], [19.0, 12.0], [14.0, 18.5]])
    out["rast_t1"], out["rast_t2"] = t1, t2
    out["rast_out"] = rasterize_seeds(SeedSpec(polygons=(t1, t2), inside_sign=-1), 24, 24)
    poly = np.array([[14.0, 14.0], [76.0, 20.0], [70.0, 76.0], [30.0, 70.0], [14.0, 50.0]])
    out["rast_b1_poly"] = poly
    out["rast_b1_out"] = rasterize_seeds(SeedSpec(polygons=(poly,), inside_sign=1), 128, 128)
    return out


def trajectory(name, image, seeds, prm, record, store=None):
    """Run the reference EvolutionRun, recording phi at the given iterations."""
    r = EvolutionRun(image, seeds, prm)
    rec = {}
    err = -1
    t0 = time.perf_counter()
    try:
        for it in sorted(record):
            r.advance(it - r.state.iteration)
            rec[it] = r.state.phi.copy()
            if r.converged:
                break
    except NumericalInstabilityError as e:
        err = e.iteration
    out = {"image": image, "iters_recorded": np.array(sorted(rec)),
           "final_iteration": np.array(r.state.iteration),
           "converged": np.array(r.converged),
           "degenerate": np.array(r.state.degenerate),
           "instability_iteration": np.array(err),
           "poly": np.stack(seeds.polygons) if len({len(p) for p in seeds.polygons}) == 1 else np.array(0),
           "inside_sign": np.array(seeds.inside_sign)}
    for it, phi in rec.items():
        if store == "hash":
            out[f"sha_{it}"] = np.array(sha(phi))
            out[f"mask_{it}"] = np.packbits(phi > 0)
        else:
            out[f"phi_{it}"] = phi
    p = prm
    out["params"] = np.array([p.dt, p.sigma2, p.ts_reg, p.reinit_period, p.reg_period,
                              p.max_iters, p.conv_check_every, p.conv_window,
                              p.model_params.sigma1, p.model_params.ts_pre,
                              p.model_params.edge_gain])
    out["model"] = np.array(p.model.value)
    out["nu"] = np.array(p.model_params.nu)
    out["mu"] = np.array(p.model_params.mu)
    print(f"{name}: iters={r.state.iteration} conv={r.converged} err={err} "
          f"{time.perf_counter() - t0:.2f}s")
    return out


def main():
    fixtures = {}
    fixtures["kernels"] = kernels_fixture()

    rng = np.random.default_rng(11)
    img_r = np.clip(two_region(48, 14, 34, 0.25, 0.7)[:, :40] + 0.05 * rng.standard_normal((48, 40)), 0, 1)
    seed_r = SeedSpec(polygons=(square(6, 8, 30, 38),), inside_sign=-1)
    fixtures["traj_region_small"] = trajectory(
        "region_small", img_r, seed_r, params(ModelKind.REGION, max_iters=25), [1, 2, 3, 10, 25])
    fixtures["traj_edge_small"] = trajectory(
        "edge_small", img_r, SeedSpec(polygons=(square(3, 3, 37, 45),), inside_sign=-1),
        params(ModelKind.EDGE, max_iters=25, sigma1=1.0, ts_pre=9), [1, 2, 3, 10, 25])
    fixtures["traj_region_field"] = trajectory(
        "region_field", img_r, seed_r,
        params(ModelKind.REGION, dt=3.0, reinit_period=0, max_iters=8), [1, 2, 4, 8])
    fixtures["traj_region_mixed"] = trajectory(
        "region_mixed", img_r, seed_r,
        params(ModelKind.REGION, dt=10.0, reinit_period=2, reg_period=3, max_iters=12),
        [1, 2, 3, 6, 12])
    fixtures["traj_edge_mixed"] = trajectory(
        "edge_mixed", img_r, SeedSpec(polygons=(square(3, 3, 37, 45),), inside_sign=-1),
        params(ModelKind.EDGE, dt=5.0, reinit_period=3, reg_period=2, max_iters=12),
        [1, 2, 3, 6, 12])
    fixtures["traj_instability"] = trajectory(
        "instability", two_region(), SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1),
        params(ModelKind.REGION, dt=1e308, reinit_period=0, max_iters=10), list(range(1, 11)), store="hash")
    fixtures["traj_degenerate"] = trajectory(
        "degenerate", np.full((32, 32), 0.5), SeedSpec(polygons=(square(0, 0, 32, 16),), inside_sign=-1),
        params(ModelKind.REGION, max_iters=3), [1, 3])
    for k, ts in enumerate([3, 5, 7]):
        img_o = np.random.default_rng(20 + k).random((33, 47))
        fixtures[f"traj_odd_ts{ts}"] = trajectory(
            f"odd_ts{ts}", img_o, SeedSpec(polygons=(square(5, 4, 30, 25),), inside_sign=1),
            params(ModelKind.REGION, ts_reg=ts, sigma2=0.8 + 0.3 * k, max_iters=15), [1, 15])
        fixtures[f"traj_odd_edge_ts{ts}"] = trajectory(
            f"odd_edge_ts{ts}", img_o, SeedSpec(polygons=(square(2, 2, 44, 30),), inside_sign=-1),
            params(ModelKind.EDGE, ts_reg=ts, ts_pre=ts, sigma1=1.2, max_iters=15), [1, 15])
    img_t = np.random.default_rng(31).random((3, 70))
    fixtures["traj_thin"] = trajectory(
        "thin", img_t, SeedSpec(polygons=(square(10, 0, 40, 2),), inside_sign=1),
        params(ModelKind.REGION, max_iters=6), [1, 6])
    a1 = two_region()
    a1_seed = SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1)
    fixtures["traj_a1"] = trajectory("a1", a1, a1_seed, params(ModelKind.REGION, max_iters=300),
                                     [300], store="hash")
    fixtures["traj_a1_cw2"] = trajectory(
        "a1_cw2", a1, a1_seed, params(ModelKind.REGION, max_iters=300, conv_check_every=5,
                                      conv_window=2), [300], store="hash")
    fixtures["traj_a1_cw1"] = trajectory(
        "a1_cw1", a1, a1_seed, params(ModelKind.REGION, max_iters=300, conv_check_every=7,
                                      conv_window=1), [300], store="hash")
    fixtures["traj_a1_edge"] = trajectory(
        "a1_edge", a1, SeedSpec(polygons=(square(28, 28, 100, 100),), inside_sign=-1),
        params(ModelKind.EDGE, max_iters=300), [300], store="hash")
    a2 = two_region(256, 48, 208, 0.41, 0.59)
    fixtures["traj_a2_edge"] = trajectory(
        "a2_edge", a2, SeedSpec(polygons=(square(36, 36, 220, 220),), inside_sign=-1),
        params(ModelKind.EDGE, max_iters=300, sigma1=1.0, ts_pre=9), [60, 300], store="hash")
    noisy = np.clip(a1 + np.random.default_rng(3).normal(0.0, 0.2, a1.shape), 0.0, 1.0)
    fixtures["traj_a5_region"] = trajectory(
        "a5_region", noisy, a1_seed, params(ModelKind.REGION, max_iters=1000), [1000], store="hash")
    fixtures["traj_a5_edge"] = trajectory(
        "a5_edge", noisy, SeedSpec(polygons=(square(20, 20, 108, 108),), inside_sign=-1),
        params(ModelKind.EDGE, max_iters=300, sigma1=1.0, ts_pre=9), [300], store="hash")

    # step() semantics: stateless single iterations from an injected +-2 state
    st = EvolutionState(phi=np.where(rasterize_seeds(seed_r, 40, 48) > 0, 2.0, -2.0))
    pe = params(ModelKind.EDGE, sigma1=1.0, ts_pre=9)
    step_out = {"image": img_r, "phi0": st.phi}
    for k in range(3):
        st = step(st, img_r, pe)
        step_out[f"phi_{k + 1}"] = st.phi
    fixtures["step_edge"] = step_out

    # the north-star configs C1 and C2 at full size (reference timing printed)
    for cfg in (scenes.config1(), scenes.config2()):
        model = ModelKind.REGION if cfg.model == "region" else ModelKind.EDGE
        prm = params(model, **cfg.params)
        seeds = SeedSpec(polygons=cfg.polygons, inside_sign=cfg.inside_sign)
        fixtures[f"traj_{cfg.name}"] = trajectory(
            cfg.name, cfg.image.astype(np.float64), seeds, prm, [cfg.iters], store="hash")
        fixtures[f"traj_{cfg.name}"]["image"] = np.array(0)   # regenerated from scenes.py

    # mean-separation (Zhang) baseline, models.py:144-162 (acceptance A4)
    zr = np.random.default_rng(41)
    zh = {}
    for k, nu in enumerate([1.5, 1.0, -0.7, 4.0]):
        img, phi = zr.random((14 + k, 19 - k)), zr.standard_normal((14 + k, 19 - k))
        v, deg = zhang_velocity(img, phi, nu)
        zh[f"img_{k}"], zh[f"phi_{k}"], zh[f"nu_{k}"] = img, phi, np.array(nu)
        zh[f"v_{k}"], zh[f"deg_{k}"] = v, np.array(deg)
    phi = rasterize_seeds(SeedSpec(polygons=(square(2, 2, 6, 6),)), 12, 12)
    v, deg = zhang_velocity(np.full((12, 12), 0.5), phi, 1.0)
    zh["img_c"], zh["phi_c"], zh["v_c"], zh["deg_c"] = np.full((12, 12), 0.5), phi, v, np.array(deg)
    fixtures["zhang"] = zh
    fixtures["traj_zhang_small"] = trajectory(
        "zhang_small", img_r, seed_r, params(ModelKind.ZHANG, max_iters=25), [1, 2, 3, 10, 25])
    fixtures["traj_zhang_nu"] = trajectory(
        "zhang_nu", img_r, SeedSpec(polygons=(square(6, 8, 30, 38),), inside_sign=1),
        params(ModelKind.ZHANG, nu=2.5, dt=6.0, max_iters=20), [1, 5, 20])
    for sign in (-1, 1):
        fixtures[f"traj_a4_{'neg' if sign < 0 else 'pos'}"] = trajectory(
            f"a4_{sign}", a1, SeedSpec(polygons=(square(28, 28, 100, 100),), inside_sign=sign),
            params(ModelKind.ZHANG, nu=1.0, max_iters=1000), [1000], store="hash")

    # curvature-regularized Chan-Vese baseline (models.py:122-141, kernels.py:98-133)
    from lsekit import curvature, signed_distance, cv_velocity, init_state
    cr = np.random.default_rng(47)
    cvu = {}
    for k in range(3):
        h, w = 13 + 5 * k, 17 + 3 * k
        m = cr.random((h, w)) > 0.6 + 0.1 * k
        m[0, 0], m[-1, -1] = True, False
        cvu[f"mask_{k}"], cvu[f"sd_{k}"] = m, signed_distance(m)
        f = cr.standard_normal((h, w))
        cvu[f"f_{k}"], cvu[f"curv_{k}"] = f, curvature(f)
        img = cr.random((h, w))
        cvu[f"img_{k}"], cvu[f"v_{k}"] = img, cv_velocity(img, f, 0.1 * (k + 1))
    a7 = two_region()
    cvu["init_a1"] = init_state(a7, SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1),
                                params(ModelKind.CHAN_VESE)).phi
    fixtures["cv_units"] = cvu
    fixtures["traj_cv_small"] = trajectory(
        "cv_small", img_r, seed_r, params(ModelKind.CHAN_VESE, max_iters=45),
        [1, 2, 19, 20, 21, 45])
    fixtures["traj_cv_a7"] = trajectory(
        "cv_a7", a7, SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1),
        params(ModelKind.CHAN_VESE, max_iters=400), [400])

    # 8-bit RGB -> grayscale of the reference loader (fileio.py:28-30, 88)
    from lsekit import fileio
    rgb = np.random.default_rng(43).integers(0, 256, size=(16, 19, 3), dtype=np.uint8)
    fixtures["luma"] = {"rgb": rgb,
                        "luma": fileio._luma(np.asarray(rgb, dtype=np.float64)) / 255.0}

    only = set(sys.argv[1:])
    for name, arrs in fixtures.items():
        if only and name not in only:
            continue
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrs)
    print("wrote", len(fixtures), "fixtures; lsekit", lsekit.__version__)


if __name__ == "__main__":
    main()
