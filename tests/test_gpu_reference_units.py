"""The reference's unit/property suite (pkg/tests/test_kernels.py,
test_grid.py, test_models.py, test_engine.py -- SURVEY §4) re-expressed
against the device-backed drop-in API, with the same tolerances."""
import warnings

import numpy as np
import pytest

import paper_1409_7474_b200 as L
from conftest import dice, square, two_region

pytestmark = pytest.mark.gpu


def direct_correlate(f, w2):
    """Brute-force same-size 2-D correlation with zero padding."""
    h, w = f.shape
    r = w2.shape[0] // 2
    out = np.zeros_like(f)
    fp = np.pad(f, r)
    for i in range(h):
        for j in range(w):
            out[i, j] = (fp[i:i + 2 * r + 1, j:j + 2 * r + 1] * w2).sum()
    return out


# ------------------------------------------------------------------ kernels
@pytest.mark.parametrize("sigma,ts", [(1.0, 9), (1.5, 5), (0.8, 3)])
def test_convolution_matches_direct_and_2d(sigma, ts):
    k = L.gaussian_kernel(sigma, ts)
    f = np.random.default_rng(ts).standard_normal((23, 19))
    got = L.convolve_same(f, k)
    w2 = np.outer(k.axis_weights, k.axis_weights)
    assert np.abs(got - direct_correlate(f, w2)).max() <= 1e-10          # test_kernels.py:61-66
    full = L.convolve_same(f, L.Kernel2D(weights=w2))
    assert np.abs(got - full).max() <= 1e-12                              # test_kernels.py:68-73


def test_convolution_linearity_and_border_attenuation():
    k = L.gaussian_kernel(1.0, 9)
    rng = np.random.default_rng(3)
    f, g = rng.standard_normal((20, 20)), rng.standard_normal((20, 20))
    lhs = L.convolve_same(2.5 * f - 0.75 * g, k)
    rhs = 2.5 * L.convolve_same(f, k) - 0.75 * L.convolve_same(g, k)
    assert np.abs(lhs - rhs).max() <= 1e-12                               # test_kernels.py:75-84
    c = L.convolve_same(np.full((20, 20), 0.6), k)
    assert np.allclose(c[4:-4, 4:-4], 0.6, atol=1e-12)                    # test_kernels.py:55-59
    assert (c[0, :] < 0.6).all() and (c[:, 0] < 0.6).all()


def test_gradients_exact_on_ramps_and_quadratics():
    yy, xx = np.mgrid[0:12, 0:15].astype(np.float64)
    fx, fy = L.gradient_central(3.0 * xx - 2.0 * yy + 1.0)
    assert np.all(fx == 3.0) and np.all(fy == -2.0)                      # test_kernels.py:93-116
    fx, fy = L.gradient_central(xx ** 2)
    assert np.array_equal(fx[:, 1:-1], 2.0 * xx[:, 1:-1]) and np.all(fy == 0.0)
    assert np.array_equal(fx[:, 0], np.ones(12)) and np.array_equal(fx[:, -1], 27.0 * np.ones(12))
    m = L.gradient_magnitude(3.0 * xx + 4.0 * yy)
    assert np.all(m == 5.0)


# --------------------------------------------------------------------- grid
def test_rasterization_matches_point_in_polygon():
    rng = np.random.default_rng(8)
    for _ in range(5):
        tri = rng.uniform(0, 30, size=(3, 2))
        try:
            got = L.rasterize_seeds(L.SeedSpec(polygons=(tri,), inside_sign=1), 30, 25)
        except L.DegenerateSeedError:
            continue
        cy, cx = np.mgrid[0:25, 0:30] + 0.5
        inside = np.zeros((25, 30), bool)
        for k in range(3):                                                # even-odd ray cast
            (x1, y1), (x2, y2) = tri[k], tri[(k + 1) % 3]
            if y1 == y2:
                continue
            cross = (y1 > cy) != (y2 > cy)
            xh = x1 + (cy - y1) * (x2 - x1) / (y2 - y1)
            inside ^= cross & (cx < xh)
        assert np.array_equal(got, np.where(inside, 1.0, -1.0))          # test_grid.py:26-32


def test_region_means_permutation_and_shift_invariance():
    rng = np.random.default_rng(5)
    img, phi = rng.random((16, 16)), rng.standard_normal((16, 16))
    cp, cm = L.region_means(img, phi)
    perm = rng.permutation(256)
    pp, pm = L.region_means(img.ravel()[perm].reshape(16, 16), phi.ravel()[perm].reshape(16, 16))
    assert abs(pp - cp) <= 1e-12 and abs(pm - cm) <= 1e-12              # test_grid.py:124-147
    sp, sm = L.region_means(img + 0.25, phi)
    assert abs(sp - (cp + 0.25)) <= 1e-12 and abs(sm - (cm + 0.25)) <= 1e-12


# ------------------------------------------------------------------- models
def test_region_velocity_affine_invariance_and_partition_swap():
    rng = np.random.default_rng(6)
    img = rng.random((24, 24))
    phi = L.convolve_same(np.where(rng.random((24, 24)) > 0.5, 1.0, -1.0), L.gaussian_kernel(1.0, 9))
    v, _ = L.region_velocity(img, phi)
    va, _ = L.region_velocity(0.5 * img + 0.1, phi)
    assert np.abs(v - va).max() <= 1e-12                                  # test_models.py:113-119
    for a, b in ((0.1, -2.0), (4.0, 2.0), (1.7, 0.3)):
        va, _ = L.region_velocity(a * img + b, phi)
        assert np.abs(v - va).max() <= 1e-12
    if not (phi == 0).any():                                              # partition swap flips
        vs, _ = L.region_velocity(img, -phi)                              # the sign (121-125)
        assert np.abs(v + vs).max() <= 1e-12


def test_edge_velocity_support_and_sign():
    rng = np.random.default_rng(7)
    img = rng.random((20, 20))
    g = L.edge_function(img, 1.0, 9)
    phi = np.ones((20, 20))
    phi[8:12, 8:12] = -1.0
    v = L.edge_velocity(g, phi)
    assert (v >= 0).all()                                                 # test_models.py:51-70
    assert np.all(v[L.gradient_magnitude(phi) == 0] == 0)


@pytest.mark.parametrize("trial", range(3))
def test_no_nan_from_finite_inputs(trial):
    rng = np.random.default_rng(trial)
    img = rng.random((16, 16))
    phi = L.binarize(rng.standard_normal((16, 16)))
    g = L.edge_function(img, 1.0, 9)
    for v in (L.edge_velocity(g, phi), L.region_velocity(img, phi)[0],
              L.zhang_velocity(img, phi, 1.0)[0]):
        assert np.isfinite(v).all()                                       # test_models.py:183-192


# ------------------------------------------------------------------- engine
def test_region_step_improves_dice():
    image, truth = two_region()
    seeds = L.SeedSpec(polygons=(square(14, 14, 76, 76),), inside_sign=-1)
    p = L.default_params(L.ModelKind.REGION)
    st = L.init_state(image, seeds, p)
    before = dice(st.phi <= 0, truth)
    for _ in range(3):
        st = L.step(st, image, p)
    assert dice(st.phi <= 0, truth) > before                             # test_engine.py:76-85
