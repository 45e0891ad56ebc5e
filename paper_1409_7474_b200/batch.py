"""Batched tiles on one GPU.

The reference evolves tiles one at a time (a worker pool of `run` calls,
engine.py:272-277).  A 1024^2 tile is far too small to fill a B200, so here
many equal-size tiles advance together: every iteration is one launch of each
fused kernel for all tiles (lse_batch_* in the C ABI).  Each tile evolves
exactly as it would alone -- same arithmetic, same per-tile reduction order --
so the results equal per-tile `run` calls bit for bit.

Tiles may be float images or 8-bit RGB arrays (H, W, 3); RGB is decoded on
the device to the reference loader's float64 luma, ((0.299 R + 0.587 G) +
0.114 B) / 255 (fileio.py:28-30, 88).
"""

from __future__ import annotations

import ctypes as C
import time
import weakref

import numpy as np

from . import _native as N
from .engine import EvolutionParams, EvolutionRun, ExtractionResult, _DeviceRun, \
    _phi0_polygons, _require_device_model
from .grid import SeedSpec, as_image
from .kernels import gaussian_kernel


def _tile_run(image, seeds: SeedSpec, params: EvolutionParams) -> EvolutionRun:
    """An EvolutionRun over a float image, or an 8-bit RGB tile decoded on the device."""
    img = np.asarray(image)
    if img.dtype == np.uint8 and img.ndim == 3 and img.shape[2] == 3:
        _require_device_model(params.model)
        run = EvolutionRun.__new__(EvolutionRun)
        run.image = np.ascontiguousarray(img)
        run.seeds = seeds
        run.params = params
        run._reg_kernel = gaussian_kernel(params.sigma2, params.ts_reg)
        init, keep = _phi0_polygons(seeds)
        run._dev = _DeviceRun(params, run.image, init, keep)
        run._version = 0
        run._snapshots = weakref.WeakSet()
        run.wall_time = 0.0
        run.trace = None
        return run
    return EvolutionRun(as_image(img), seeds, params)


class TileBatch:
    """Advance several EvolutionRuns of one tile size together.

    The runs must share size and evolution parameters (model, image and seeds
    may differ) and stay on the binary-state path (reinit_period =
    reg_period = 1).  Each run remains usable on its own afterwards.
    """

    def __init__(self, runs):
        self.runs = list(runs)
        if not self.runs:
            raise ValueError("empty batch")
        if any(r.trace is not None for r in self.runs):
            raise ValueError("runs with a contour trace advance on their own")
        handles = (C.c_void_p * len(self.runs))(*[r._dev.h.value for r in self.runs])
        h = C.c_void_p()
        N.check(N.lib.lse_batch_create(C.byref(h), handles, len(self.runs)))
        self.h = h
        self._fin = weakref.finalize(self, N.lib.lse_batch_destroy, h)

    def advance(self, n_steps: int):
        if n_steps < 0:
            raise ValueError("n_steps must be >= 0")
        for r in self.runs:
            r._before_mutation()
        st = (N.LseStatus * len(self.runs))()
        t0 = time.perf_counter()
        N.check(N.lib.lse_batch_advance(self.h, int(n_steps), st))
        dt = time.perf_counter() - t0
        for r in self.runs:
            r.wall_time += dt
        return [r.state for r in self.runs]

    def close(self):
        self._fin()


def run_tiles(images, seeds, params) -> list[ExtractionResult]:
    """`run` (engine.py:272-277) for every tile, advanced as one batch.

    images: a sequence (or array) of equal-size tiles, float (H, W) or uint8
    (H, W, 3); seeds / params: one per tile or a single shared value.
    """
    n = len(images)
    seeds = list(seeds) if isinstance(seeds, (list, tuple)) else [seeds] * n
    params = list(params) if isinstance(params, (list, tuple)) else [params] * n
    if len(seeds) != n or len(params) != n:
        raise ValueError("one seed spec and one parameter set per tile")
    runs = [_tile_run(images[k], seeds[k], params[k]) for k in range(n)]
    batch = TileBatch(runs)
    batch.advance(max(p.max_iters for p in params))
    out = [r.result() for r in runs]
    batch.close()
    return out
