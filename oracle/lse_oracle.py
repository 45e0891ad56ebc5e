"""CPU oracle for the LSE hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference algorithm
(`lsekit` 0.1.0, /root/reference/pkg/src/lsekit).  It is the *checker*:
only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
may import it.  The product package (`paper_1409_7474_b200`) never imports
anything under `oracle/`; it fails loudly when its CUDA library is missing.

Parity is pinned: `tests/golden/make_golden.py` runs the reference itself
(importable in the build container) and commits its outputs; the
`-m "not gpu"` tests assert this restatement reproduces them bit-for-bit.

Third-party arithmetic the reference reaches, restated here:
* scipy 1.18.1 `ndimage.correlate1d` (symmetric-kernel branch of scipy's
  NI_Correlate1D: out = x[0]*w[0]; then for distance d = r..1:
  out += (x[-d] + x[+d]) * w[d]); verified bit-exact against scipy here.
* numpy 2.3.5 `np.gradient` (edge_order=1) and `ndarray.mean` (pairwise
  summation: 8-way unrolled blocks of <=128, recursive halving with the
  split rounded down to a multiple of 8).
* glibc (>=2.35) `hypot`, which `np.hypot` calls on x86-64: the non-FMA
  Borges correction kernel.  np.hypot is used directly here; the same
  algorithm is restated in oracle/lse_oracle.c and in the CUDA fallback.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

REGION = "region"
EDGE = "edge"
ZHANG = "zhang"
CV = "cv"
DT_STABILITY_LIMIT = 25.0          # engine.py:26


class OracleInstability(RuntimeError):
    """engine.py:29-37 -- non-finite level-set values at `iteration`."""

    def __init__(self, iteration):
        super().__init__(f"numerical instability at iteration {iteration}")
        self.iteration = iteration


# --------------------------------------------------------------------------
# kernels.py
# --------------------------------------------------------------------------

def gaussian_weights(sigma: float, ts: int) -> np.ndarray:
    """kernels.py:50-64 -- sampled, renormalized 1-D Gaussian of odd size."""
    if sigma <= 0 or ts < 1 or ts % 2 == 0:
        raise ValueError("bad gaussian parameters")
    c = (ts - 1) / 2.0
    x = np.arange(ts, dtype=np.float64) - c
    w1 = np.exp(-(x * x) / (2.0 * sigma * sigma))
    w1 /= w1.sum()
    return w1


def correlate1d_same(f: np.ndarray, w: np.ndarray, axis: int) -> np.ndarray:
    """kernels.py:72-76 (scipy.ndimage.correlate1d, mode='constant', cval=0).

    Symmetric odd kernel: out = x[0]*w[c], then for d = r..1 (outermost
    pair first) out += (x[-d] + x[+d]) * w[c-d].  Zero padding outside.
    """
    f = np.asarray(f, dtype=np.float64)
    g = np.moveaxis(f, axis, -1)
    n = g.shape[-1]
    ts = len(w)
    r = ts // 2
    pad = np.zeros(g.shape[:-1] + (n + 2 * r,))
    pad[..., r:r + n] = g
    out = pad[..., r:r + n] * w[r]
    for d in range(r, 0, -1):
        out = out + (pad[..., r - d:r - d + n] + pad[..., r + d:r + d + n]) * w[r - d]
    return np.ascontiguousarray(np.moveaxis(out, -1, axis))


def convolve_same(f: np.ndarray, w: np.ndarray) -> np.ndarray:
    """kernels.py:67-78 -- separable path: axis 0 (rows) then axis 1."""
    return correlate1d_same(correlate1d_same(f, w, 0), w, 1)


def gradient_central(f: np.ndarray):
    """kernels.py:81-90 (np.gradient, unit spacing, edge_order=1).

    Interior (f[i+1]-f[i-1])/2.0, one-sided f[1]-f[0] / f[n-1]-f[n-2] at
    the first/last row and column.  Returns (fx, fy).
    """
    f = np.asarray(f, dtype=np.float64)
    if f.ndim != 2 or f.shape[0] < 2 or f.shape[1] < 2:
        raise ValueError("gradient needs at least a 2x2 field")
    fy = np.empty_like(f)
    fx = np.empty_like(f)
    fy[1:-1, :] = (f[2:, :] - f[:-2, :]) / 2.0
    fy[0, :] = (f[1, :] - f[0, :]) / 1.0
    fy[-1, :] = (f[-1, :] - f[-2, :]) / 1.0
    fx[:, 1:-1] = (f[:, 2:] - f[:, :-2]) / 2.0
    fx[:, 0] = (f[:, 1] - f[:, 0]) / 1.0
    fx[:, -1] = (f[:, -1] - f[:, -2]) / 1.0
    return fx, fy


def gradient_magnitude(f: np.ndarray) -> np.ndarray:
    """kernels.py:93-95 -- hypot of the central-difference gradient."""
    fx, fy = gradient_central(f)
    return np.hypot(fx, fy)


def glibc_hypot(x: float, y: float) -> float:
    """Scalar restatement of glibc's non-FMA hypot (what np.hypot calls)."""
    if not (math.isfinite(x) and math.isfinite(y)):
        if math.isinf(x) or math.isinf(y):
            return math.inf
        return x + y
    x, y = abs(x), abs(y)
    ax, ay = (y, x) if x < y else (x, y)
    scale, large, tiny, eps = 2.0 ** -600, 2.0 ** 511, 2.0 ** -511, 2.0 ** -54

    def kern(ax, ay):
        h = math.sqrt(ax * ax + ay * ay)
        if h <= 2.0 * ay:
            delta = h - ay
            t1 = ax * (2.0 * delta - ax)
            t2 = (delta - 2.0 * (ax - ay)) * delta
        else:
            delta = h - ax
            t1 = 2.0 * delta * (ax - 2.0 * ay)
            t2 = (4.0 * delta - ay) * ay + delta * delta
        return h - (t1 + t2) / (2.0 * h)

    if ax > large:
        if ay <= ax * eps:
            return ax + ay
        return kern(ax * scale, ay * scale) / scale
    if ay < tiny:
        if ax >= ay / eps:
            return ax + ay
        return kern(ax / scale, ay / scale) * scale
    if ay <= ax * eps:
        return ax + ay
    return kern(ax, ay)


# --------------------------------------------------------------------------
# grid.py
# --------------------------------------------------------------------------

def binarize(phi: np.ndarray) -> np.ndarray:
    """grid.py:96-99 -- +1 where phi > 0, -1 where phi <= 0."""
    return np.where(np.asarray(phi, dtype=np.float64) > 0.0, 1.0, -1.0)


def region_means(image: np.ndarray, phi: np.ndarray):
    """grid.py:102-118 -- means over phi >= 0 (ties positive) and phi < 0.

    Returns None for an empty side (DegeneratePartitionError in the
    reference).  numpy's pairwise `mean` is the reference's own arithmetic.
    """
    pos = phi >= 0.0
    n_pos = int(pos.sum())
    if n_pos == 0 or n_pos == pos.size:
        return None
    return float(image[pos].mean()), float(image[~pos].mean())


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's pairwise float64 summation (what `mean` uses), restated."""
    n = len(a)
    if n < 8:
        res = 0.0
        for i in range(n):
            res += float(a[i])
        return res
    if n <= 128:
        r = [float(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def polygon_mask(poly: np.ndarray, width: int, height: int) -> np.ndarray:
    """grid.py:58-73 -- even-odd ray casting at pixel centres."""
    px = np.arange(width, dtype=np.float64) + 0.5
    py = np.arange(height, dtype=np.float64) + 0.5
    cx, cy = np.meshgrid(px, py)
    inside = np.zeros((height, width), dtype=bool)
    n = poly.shape[0]
    for i in range(n):
        x1, y1 = poly[i]
        x2, y2 = poly[(i + 1) % n]
        if y1 == y2:
            continue
        crosses = (y1 > cy) != (y2 > cy)
        x_hit = x1 + (cy - y1) * (x2 - x1) / (y2 - y1)
        inside ^= crosses & (cx < x_hit)
    return inside


def rasterize_seeds(polygons, inside_sign: int, width: int, height: int) -> np.ndarray:
    """grid.py:76-93 -- union of polygon interiors gets inside_sign.

    Returns None when the union is empty or covers the grid
    (DegenerateSeedError in the reference).
    """
    inside = np.zeros((height, width), dtype=bool)
    for poly in polygons:
        inside |= polygon_mask(np.asarray(poly, dtype=np.float64), width, height)
    if not inside.any() or inside.all():
        return None
    s = float(inside_sign)
    return np.where(inside, s, -s)


# --------------------------------------------------------------------------
# models.py
# --------------------------------------------------------------------------

def edge_function(image: np.ndarray, sigma1: float, ts_pre: int,
                  gain: float = 255.0) -> np.ndarray:
    """models.py:71-81 -- 1/(1 + (gain fx)^2 + (gain fy)^2) of G*I."""
    smoothed = convolve_same(np.asarray(image, dtype=np.float64),
                             gaussian_weights(sigma1, ts_pre))
    fx, fy = gradient_central(smoothed)
    return 1.0 / (1.0 + (gain * fx) ** 2 + (gain * fy) ** 2)


def edge_velocity(g: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """models.py:84-90 -- g * |grad phi|."""
    return g * gradient_magnitude(phi)


def region_velocity(image: np.ndarray, phi: np.ndarray):
    """models.py:101-119 -- (D / max|D|) * |grad phi|, D=(c+-c-)(2I-c+-c-)."""
    means = region_means(image, phi)
    if means is None:
        return np.zeros_like(phi), True
    c_plus, c_minus = means
    data = (c_plus - c_minus) * (2.0 * image - c_plus - c_minus)
    peak = float(np.abs(data).max())
    if peak == 0.0:
        return np.zeros_like(phi), True
    return (data / peak) * gradient_magnitude(phi), False


def curvature(phi: np.ndarray, eps_guard: float = 1e-10) -> np.ndarray:
    """kernels.py:98-115 -- (pxx py^2 - 2 px py pxy + pyy px^2) / (px^2+py^2+eps)^1.5."""
    px, py = gradient_central(phi)
    pxx = np.gradient(px, axis=1)
    pxy = np.gradient(px, axis=0)
    pyy = np.gradient(py, axis=0)
    num = pxx * py * py - 2.0 * px * py * pxy + pyy * px * px
    den = np.power(px * px + py * py + eps_guard, 1.5)
    return num / den


def squared_edt(target: np.ndarray) -> np.ndarray:
    """Exact squared Euclidean distance to the nearest True pixel (the quantity
    scipy's distance_transform_edt takes the root of): per column the distance
    to the nearest target, then per row min_x' g(x') + (x - x')^2, all in
    integers."""
    h, w = target.shape
    inf = np.int64(1) << 40
    ys = np.arange(h, dtype=np.int64)
    g = np.full((h, w), inf, dtype=np.int64)
    for x in range(w):
        t = np.nonzero(target[:, x])[0]
        if len(t):
            g[:, x] = np.abs(ys[:, None] - t[None, :]).min(axis=1) ** 2
    xs = np.arange(w, dtype=np.int64)
    return (g[:, None, :] + (xs[None, :, None] - xs[None, None, :]) ** 2).min(axis=2)


def signed_distance(mask: np.ndarray) -> np.ndarray:
    """kernels.py:118-133 -- edt(~obj) - edt(obj): positive outside, centre to
    centre, sqrt of integer squared distances."""
    obj = np.asarray(mask, dtype=bool)
    d_out = np.sqrt(squared_edt(obj).astype(np.float64))
    d_in = np.sqrt(squared_edt(~obj).astype(np.float64))
    d_out[obj] = 0.0
    d_in[~obj] = 0.0
    return d_out - d_in


def cv_velocity(image: np.ndarray, phi: np.ndarray, mu: float, eps_guard: float = 1e-10):
    """models.py:122-141 -- [(c+ - c-)(2I - c+ - c-) + mu kappa] |grad phi|."""
    means = region_means(image, phi)
    if means is None:
        data = np.zeros_like(phi)
    else:
        c_plus, c_minus = means
        data = (c_plus - c_minus) * (2.0 * image - c_plus - c_minus)
    if mu != 0.0:
        data = data + mu * curvature(phi, eps_guard)
    return data * gradient_magnitude(phi)


def region_velocity_bands(image: np.ndarray, phi: np.ndarray):
    """Multi-band region data term -- a restatement, the
    reference is single-band (grid.py:27-28): D = sum_k (c+_k - c-_k)(2 I_k -
    c+_k - c-_k), bands accumulated in order, then models.py:109-119.  With one
    band this is region_velocity exactly (its parity is pinned by that)."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim == 2:
        image = image[None]
    pos = phi >= 0.0
    n_pos = int(pos.sum())
    if n_pos == 0 or n_pos == pos.size:
        return np.zeros_like(phi), True
    data = None
    for band in image:
        c_plus, c_minus = float(band[pos].mean()), float(band[~pos].mean())
        term = (c_plus - c_minus) * (2.0 * band - c_plus - c_minus)
        data = term if data is None else data + term
    peak = float(np.abs(data).max())
    if peak == 0.0:
        return np.zeros_like(phi), True
    return (data / peak) * gradient_magnitude(phi), False


def zhang_velocity(image: np.ndarray, phi: np.ndarray, nu: float):
    """models.py:144-162 -- nu * ((I - m) / max|I - m|) * |grad phi|, m = (c+ + c-)/2."""
    means = region_means(image, phi)
    if means is None:
        return np.zeros_like(phi), True
    c_plus, c_minus = means
    centered = image - 0.5 * (c_plus + c_minus)
    peak = float(np.abs(centered).max())
    if peak == 0.0:
        return np.zeros_like(phi), True
    return nu * (centered / peak) * gradient_magnitude(phi), False


# --------------------------------------------------------------------------
# engine.py:280-294 extract_contours -> skimage.measure.find_contours
# (scikit-image >= 0.20, pkg/pyproject.toml:13; absent here, so restated from
# its published algorithm: marching-squares segments per 2x2 square in
# row-major order, then the dict-based endpoint join).  Parity with
# scikit-image itself is unpinned; the reference's own contour tests
# (tests/test_engine.py:202-228) and hand-derived cases pin this restatement.
# --------------------------------------------------------------------------

# case -> (from, to) edge pairs; edges 0 top, 1 bottom, 2 left, 3 right;
# saddles 6 / 9 keep the low values connected (fully_connected='low')
_MS_CASES = {1: ((0, 2),), 2: ((3, 0),), 3: ((3, 2),), 4: ((2, 1),), 5: ((0, 1),),
             6: ((3, 0), (2, 1)), 7: ((3, 1),), 8: ((1, 3),), 9: ((0, 2), (1, 3)),
             10: ((1, 0),), 11: ((1, 2),), 12: ((2, 3),), 13: ((0, 3),), 14: ((2, 0),)}


def _ms_fraction(f, t):
    with np.errstate(divide="ignore", invalid="ignore"):
        q = (0.0 - f) / (t - f)
    return np.where(t == f, 0.0, q)


def contour_segments(phi: np.ndarray):
    """Oriented segments ((r, c), (r, c)) of level 0, in square order."""
    a = np.asarray(phi, dtype=np.float64)
    ul, ur, ll, lr = a[:-1, :-1], a[:-1, 1:], a[1:, :-1], a[1:, 1:]
    cs = ((ul > 0).astype(np.int64) + 2 * (ur > 0) + 4 * (ll > 0) + 8 * (lr > 0))
    nan = np.isnan(ul) | np.isnan(ur) | np.isnan(ll) | np.isnan(lr)
    r0, c0 = np.meshgrid(np.arange(a.shape[0] - 1, dtype=np.float64),
                         np.arange(a.shape[1] - 1, dtype=np.float64), indexing="ij")
    pts = (
        (r0, c0 + _ms_fraction(ul, ur)),        # top
        (r0 + 1.0, c0 + _ms_fraction(ll, lr)),  # bottom
        (r0 + _ms_fraction(ul, ll), c0),        # left
        (r0 + _ms_fraction(ur, lr), c0 + 1.0),  # right
    )
    segs = []
    rows, cols = np.nonzero((cs != 0) & (cs != 15) & ~nan)
    for i, j in zip(rows.tolist(), cols.tolist()):
        for e0, e1 in _MS_CASES[int(cs[i, j])]:
            segs.append(((float(pts[e0][0][i, j]), float(pts[e0][1][i, j])),
                         (float(pts[e1][0][i, j]), float(pts[e1][1][i, j]))))
    return segs


def assemble_contours(segments):
    """Join oriented segments into polylines (the published dict algorithm)."""
    from collections import deque
    index = 0
    contours, starts, ends = {}, {}, {}
    for p0, p1 in segments:
        if p0 == p1:
            continue
        tail, tail_num = starts.pop(p1, (None, None))
        head, head_num = ends.pop(p0, (None, None))
        if tail is not None and head is not None:
            if tail is head:
                head.append(p1)
            elif tail_num > head_num:
                head.extend(tail)
                contours.pop(tail_num, None)
                starts[head[0]] = (head, head_num)
                ends[head[-1]] = (head, head_num)
            else:
                tail.extendleft(reversed(head))
                starts.pop(head[0], None)
                contours.pop(head_num, None)
                starts[tail[0]] = (tail, tail_num)
                ends[tail[-1]] = (tail, tail_num)
        elif tail is None and head is None:
            c = deque((p0, p1))
            contours[index] = c
            starts[p0] = (c, index)
            ends[p1] = (c, index)
            index += 1
        elif head is None:
            tail.appendleft(p0)
            starts[p0] = (tail, tail_num)
        else:
            head.append(p1)
            ends[p1] = (head, head_num)
    return [np.array(c) for _, c in sorted(contours.items())]


def extract_contours(phi: np.ndarray):
    """engine.py:280-294: (x, y) = (col + 0.5, row + 0.5) polylines."""
    phi = np.asarray(phi, dtype=np.float64)
    if not ((phi > 0).any() and (phi < 0).any()):
        return []
    out = []
    for c in assemble_contours(contour_segments(phi)):
        out.append(np.stack([c[:, 1] + 0.5, c[:, 0] + 0.5], axis=1))
    return out


# --------------------------------------------------------------------------
# engine.py
# --------------------------------------------------------------------------

@dataclass
class OracleParams:
    """engine.py:40-81 / models.py:44-68 (validation lives in the product)."""
    model: str = REGION
    dt: float = 15.0
    sigma2: float = 1.0
    ts_reg: int = 9
    reinit_period: int = 1
    reg_period: int = 1
    max_iters: int = 1000
    conv_check_every: int = 10
    conv_window: int = 3
    sigma1: float = 1.0
    ts_pre: int = 9
    edge_gain: float = 255.0
    nu: float = 1.0
    mu: float = 0.1


def advance_once(phi, iteration, image, p: OracleParams, g, w_reg):
    """engine.py:148-174 -- update, finiteness, reinit, regularize, guard."""
    if p.model == EDGE:
        v, degenerate = edge_velocity(g, phi), False
    elif p.model == ZHANG:
        v, degenerate = zhang_velocity(image, phi, p.nu)
    elif p.model == CV:
        v, degenerate = cv_velocity(image, phi, p.mu), False
    elif image.ndim == 3:
        v, degenerate = region_velocity_bands(image, phi)
    else:
        v, degenerate = region_velocity(image, phi)
    out = phi + p.dt * v
    n = iteration + 1
    if np.isfinite(out).all():
        if p.reinit_period > 0 and n % p.reinit_period == 0:
            if p.model == CV:                        # engine.py:161-165
                b = binarize(out)
                if (b > 0).any() and (b < 0).any():
                    out = -signed_distance(b > 0)
            else:
                out = binarize(out)
        if n % p.reg_period == 0:
            out = convolve_same(out, w_reg)
    if not np.isfinite(out).all():
        raise OracleInstability(n)
    return out, n, degenerate


class OracleRun:
    """engine.py:193-269 -- resumable driver with checkpoint convergence."""

    def __init__(self, image, phi0, p: OracleParams, iteration=0, trace=False):
        self.image = np.asarray(image, dtype=np.float64)
        self.p = p
        self.phi = np.asarray(phi0, dtype=np.float64)
        self.iteration = iteration
        self.converged = False
        self.degenerate = False
        self.w_reg = gaussian_weights(p.sigma2, p.ts_reg)
        self.g = (edge_function(self.image, p.sigma1, p.ts_pre, p.edge_gain)
                  if p.model == EDGE else None)
        self.checkpoints = []
        self.trace = [(0, extract_contours(self.phi))] if trace else None   # engine.py:214-216

    def step_once(self):
        p = self.p
        phi, n, degenerate = advance_once(self.phi, self.iteration, self.image,
                                          p, self.g, self.w_reg)
        converged = False
        if n % p.conv_check_every == 0:
            self.checkpoints.append(phi > 0)
            if len(self.checkpoints) > p.conv_window:
                self.checkpoints.pop(0)
            if len(self.checkpoints) == p.conv_window and all(
                    np.array_equal(self.checkpoints[-1], m)
                    for m in self.checkpoints[:-1]):
                converged = True
            if self.trace is not None:                      # engine.py:237-238
                self.trace.append((n, extract_contours(phi)))
        self.phi, self.iteration = phi, n
        self.converged = converged
        self.degenerate = self.degenerate or degenerate

    def advance(self, n_steps):
        for _ in range(n_steps):
            if self.converged or self.iteration >= self.p.max_iters:
                break
            self.step_once()
        return self

    def mask(self, inside_sign):
        return (self.phi > 0) if inside_sign > 0 else (self.phi <= 0)


def run_fixed(image, phi0, p: OracleParams, n_iters: int):
    """Fixed-iteration run (conv_check_every = n+1 semantics)."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        r = OracleRun(image, phi0, p)
        r.advance(n_iters)
    return r
