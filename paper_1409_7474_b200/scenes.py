"""Seeded synthetic scenes standing in for BASELINE.json's five configs.

The paper's Google-Maps images are not available, so the
benchmark and parity suites use these generators.
Images are generated in float64, clipped to [0, 1] and stored as float32;
the reference receives ``I32.astype(float64)``, which is exact, so both
sides see identical inputs.  Seeds: numpy PCG64, seed = 1000*config + k.

Every generator returns a ``Scene``: the float32 image, the seed polygon(s)
with their interior sign, and the evolution parameters of the config.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Scene:
    name: str
    image: np.ndarray                  # float32 (H, W), values in [0, 1]
    polygons: tuple                    # seed polygons in (x, y) pixel coords
    inside_sign: int
    params: dict                       # kwargs for default_params(model, ...)
    model: str                         # "region" | "edge"
    iters: int
    extra: dict = field(default_factory=dict)


def box_polygon(x0, y0, x1, y1):
    return np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], dtype=np.float64)


def _fill_rects(img, rng, n, side_lo, side_hi, mean, std):
    h, w = img.shape
    for _ in range(n):
        sw = int(rng.integers(side_lo, side_hi + 1))
        sh = int(rng.integers(side_lo, side_hi + 1))
        x = int(rng.integers(0, max(1, w - sw)))
        y = int(rng.integers(0, max(1, h - sh)))
        block = img[y:y + sh, x:x + sw]
        block[...] = mean + std * rng.standard_normal(block.shape)


def config1(size=256):
    """C1: 256^2 single band, 5 roofs on N(0.30,0.05), region, dt=100, 5x5."""
    rng = np.random.default_rng(1000)
    img = 0.30 + 0.05 * rng.standard_normal((size, size))
    _fill_rects(img, rng, 5, 20, 80, 0.75, 0.05)
    img = np.clip(img, 0.0, 1.0).astype(np.float32)
    m = (size - 200) // 2
    return Scene("C1", img, (box_polygon(m, m, m + 200, m + 200),), +1,
                 dict(dt=100.0, sigma2=1.0, ts_reg=5, max_iters=200,
                      conv_check_every=201), "region", 200)


def _value_noise(rng, n, octaves=4, base=8):
    out = np.zeros((n, n))
    amp = 1.0
    for o in range(octaves):
        cells = base * (2 ** o)
        grid = rng.random((cells + 1, cells + 1))
        t = np.linspace(0.0, cells, n, endpoint=False)
        i0 = np.floor(t).astype(int)
        f = t - i0
        f = f * f * (3.0 - 2.0 * f)
        a = grid[i0][:, i0]
        b = grid[i0][:, i0 + 1]
        c = grid[i0 + 1][:, i0]
        d = grid[i0 + 1][:, i0 + 1]
        fx = f[None, :]
        fy = f[:, None]
        out += amp * ((a * (1 - fx) + b * fx) * (1 - fy) + (c * (1 - fx) + d * fx) * fy)
        amp *= 0.5
    return out


def _draw_polyline(img, pts, width, value):
    h, w = img.shape
    r = width / 2.0
    for (x1, y1), (x2, y2) in zip(pts[:-1], pts[1:]):
        xa, xb = int(max(0, np.floor(min(x1, x2) - r))), int(min(w, np.ceil(max(x1, x2) + r) + 1))
        ya, yb = int(max(0, np.floor(min(y1, y2) - r))), int(min(h, np.ceil(max(y1, y2) + r) + 1))
        if xa >= xb or ya >= yb:
            continue
        yy, xx = np.mgrid[ya:yb, xa:xb]
        px, py = xx + 0.5, yy + 0.5
        dx, dy = x2 - x1, y2 - y1
        L2 = dx * dx + dy * dy
        tt = np.clip(((px - x1) * dx + (py - y1) * dy) / max(L2, 1e-12), 0.0, 1.0)
        d2 = (px - (x1 + tt * dx)) ** 2 + (py - (y1 + tt * dy)) ** 2
        sel = d2 <= r * r
        img[ya:yb, xa:xb][sel] = value[ya:yb, xa:xb][sel]


def config2(size=1024):
    """C2: 1024^2 road scene on 4-octave value noise, edge model, 500 its."""
    rng = np.random.default_rng(2000)
    noise = _value_noise(rng, size)
    noise = (noise - noise.mean()) / noise.std()
    img = 0.4 + 0.08 * noise
    road_val = 0.65 + 0.03 * rng.standard_normal((size, size))
    for _ in range(6):
        nv = int(rng.integers(3, 7))
        pts = rng.uniform(0, size, size=(nv, 2))
        width = float(rng.uniform(8, 20))
        _draw_polyline(img, pts, width, road_val)
    img = np.clip(img, 0.0, 1.0).astype(np.float32)
    m = (size - 900) // 2
    return Scene("C2", img, (box_polygon(m, m, m + 900, m + 900),), -1,
                 dict(dt=15.0, sigma2=1.0, ts_reg=9, sigma1=1.5, ts_pre=9,
                      edge_gain=255.0, max_iters=500, conv_check_every=501),
                 "edge", 500)


def config3(size=4096, iters=1000, n_shapes=400):
    """C3: 4-band (B, G, R, NIR) scene, float32 (4, H, W): background
    N((.25, .30, .28, .45), .05), n_shapes rectangles / convex polygons of
    10-120 px with N((.60, .62, .65, .35), .04); region model on the vector
    data term, sigma2 1.0 (9 taps), dt 15; initial state a +-1 checkerboard of
    64 x 64 cells (extra["signs"], int8), SURVEY section 8d."""
    rng = np.random.default_rng(3000)
    bg = np.array([0.25, 0.30, 0.28, 0.45])
    fg = np.array([0.60, 0.62, 0.65, 0.35])
    img = bg[:, None, None] + 0.05 * rng.standard_normal((4, size, size))
    yy, xx = np.mgrid[0:size, 0:size]
    n_shapes = max(1, int(round(n_shapes * (size / 4096.0) ** 2)))
    for s in range(n_shapes):
        w, h = (int(v) for v in rng.integers(10, 121, size=2))
        x0 = int(rng.integers(0, max(1, size - w)))
        y0 = int(rng.integers(0, max(1, size - h)))
        vals = fg[:, None, None] + 0.04 * rng.standard_normal((4, h, w))
        if s % 2 == 0:                               # rectangle
            img[:, y0:y0 + h, x0:x0 + w] = vals
        else:                                        # convex polygon: an inscribed ellipse
            cy, cx = h / 2.0, w / 2.0
            m = ((yy[:h, :w] + 0.5 - cy) / cy) ** 2 + ((xx[:h, :w] + 0.5 - cx) / cx) ** 2 <= 1.0
            sub = img[:, y0:y0 + h, x0:x0 + w]
            sub[:, m] = vals[:, m]
    img = np.clip(img, 0.0, 1.0).astype(np.float32)
    cells = (yy // 64 + xx // 64) % 2
    signs = np.where(cells == 0, 1, -1).astype(np.int8)
    return Scene("C3", img, (), 1, dict(dt=15.0, sigma2=1.0, ts_reg=9, max_iters=iters,
                                        conv_check_every=iters + 1), "region", iters,
                 extra=dict(signs=signs))


def config4_tile(k, size=1024, iters=300):
    """C4 tile k: 8-bit RGB (H, W, 3) urban tile; even tiles region with +inside
    seeds, odd tiles edge (sigma1 1.0, gain 255) with -inside seeds; centred
    900^2 seed box.  Background U[40,90], rectangles
    U[150,220], 10-16 px roads U[100,140], N(0, 6) noise, clipped to 0..255."""
    rng = np.random.default_rng(4000 + k)
    img = np.empty((size, size, 3), dtype=np.float64)
    img[...] = rng.uniform(40, 90, size=3)
    for _ in range(int(rng.integers(10, 25))):
        sw, sh = (int(v) for v in rng.integers(24, max(25, size // 5), size=2))
        x = int(rng.integers(0, max(1, size - sw)))
        y = int(rng.integers(0, max(1, size - sh)))
        img[y:y + sh, x:x + sw] = rng.uniform(150, 220, size=3)
    for _ in range(int(rng.integers(2, 4))):
        nv = int(rng.integers(2, 5))
        pts = rng.uniform(0, size, size=(nv, 2))
        width = float(rng.uniform(10, 16))
        col = rng.uniform(100, 140, size=3)
        for ch in range(3):
            _draw_polyline(img[..., ch], pts, width, np.full((size, size), col[ch]))
    img += rng.normal(0.0, 6.0, size=img.shape)
    img = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    m = (size - min(900, size - 2)) // 2
    region = k % 2 == 0
    params = dict(dt=15.0, sigma2=1.0, ts_reg=9, max_iters=iters, conv_check_every=iters + 1)
    if not region:
        params.update(sigma1=1.0, ts_pre=9, edge_gain=255.0)
    return Scene("C4", img, (box_polygon(m, m, size - m, size - m),), 1 if region else -1,
                 params, "region" if region else "edge", iters, extra=dict(tile=k))


def luma(rgb):
    """The reference loader's grayscale of an 8-bit RGB array (fileio.py:28-30,
    88): ((0.299 R + 0.587 G) + 0.114 B) / 255 in float64."""
    x = np.asarray(rgb, dtype=np.float64)
    return (0.299 * x[..., 0] + 0.587 * x[..., 1] + 0.114 * x[..., 2]) / 255.0


def config5(size=32768, n_rects=20000, iters=500, seed_offset=0, rows=None):
    """C5: large panchromatic scene, 20000 rects 8-64 px, region, sigma 1.5.

    ``size``/``n_rects`` may be scaled down together (same object density)
    for parity crops: n_rects_crop = n_rects * (size/32768)^2.  ``rows =
    (y0, y1)`` generates only those image rows (a row strip of a multi-GPU
    run); the pixels are identical to the same rows of the full image: the
    background noise comes in fixed row blocks with their own seeded
    streams, the rectangles from one stream drawn completely by every caller.
    """
    y0, y1 = (0, size) if rows is None else (int(rows[0]), int(rows[1]))
    base = 5000 + seed_offset
    img = np.empty((y1 - y0, size), dtype=np.float32)
    block = max(1, (1 << 24) // size)
    for k, y in enumerate(range(0, size, block)):
        ye = min(size, y + block)
        if ye <= y0 or y >= y1:
            continue
        z = np.random.default_rng([base, 1, k]).standard_normal((ye - y, size),
                                                                 dtype=np.float32)
        a, b = max(y, y0), min(ye, y1)
        img[a - y0:b - y0] = np.float32(0.3) + np.float32(0.05) * z[a - y:b - y]
    rng = np.random.default_rng([base, 2])
    for _ in range(n_rects):
        sw = int(rng.integers(8, 65))
        sh = int(rng.integers(8, 65))
        x = int(rng.integers(0, max(1, size - sw)))
        y = int(rng.integers(0, max(1, size - sh)))
        vals = np.float32(0.7) + np.float32(0.05) * rng.standard_normal((sh, sw),
                                                                          dtype=np.float32)
        a, b = max(y, y0), min(y + sh, y1)
        if a < b:
            img[a - y0:b - y0, x:x + sw] = vals[a - y:b - y]
    np.clip(img, 0.0, 1.0, out=img)
    m = size // 16
    return Scene("C5", img, (box_polygon(m, m, size - m, size - m),), -1,
                 dict(dt=15.0, sigma2=1.5, ts_reg=9, max_iters=iters,
                      conv_check_every=iters + 1), "region", iters,
                 extra=dict(n_rects=n_rects, rows=(y0, y1)))


def config5_crop(size=4096, iters=500):
    """C5 at reduced size, same object density (parity crop)."""
    n = max(1, int(round(20000 * (size / 32768.0) ** 2)))
    return config5(size=size, n_rects=n, iters=iters, seed_offset=size)
