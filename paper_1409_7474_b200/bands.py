"""Multi-band images: the region model with a vector data term.

The reference is single-band (as_field rejects non-2-D input, grid.py:24-31).
C3 extends the region evolution to K <= 4 bands with

    D = sum_k (c+_k - c-_k) (2 I_k - c+_k - c-_k)

(bands accumulated in order; c+_k / c-_k the band means over phi >= 0 /
phi < 0), then the reference's own normalization v = D / max|D| * |grad phi|
(models.py:109-119).  With one band this is the region model exactly, which
pins the restatement (oracle/lse_oracle.py: region_velocity_bands).

On the device each iteration adds one pass over the bands after the
partition: per-band means, then D of every pixel in fp64 (stored as the fp32
data plane of the fused kernels) and its peak; the fused update then runs the
single-band region kernels with vf = (dt/2) D / peak.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _native as N
from .engine import (EvolutionParams, EvolutionRun, ModelKind, _DeviceRun, _native_params,
                     _phi0_polygons)
from .grid import SeedSpec, DegenerateSeedError
from .kernels import gaussian_kernel


def as_bands(bands) -> np.ndarray:
    """(K, H, W) float image, 1 <= K <= 4, finite (grid.py:24-31 per band)."""
    b = np.asarray(bands)
    if b.ndim == 2:
        b = b[None]
    if b.ndim != 3 or not 1 <= b.shape[0] <= 4:
        raise ValueError("expected a (K, H, W) image with 1 <= K <= 4 bands")
    if b.dtype not in (np.float32, np.float64):
        b = b.astype(np.float64)
    if not np.isfinite(b).all():
        raise ValueError("image contains non-finite values")
    return np.ascontiguousarray(b)


class _BandDeviceRun(_DeviceRun):
    def __init__(self, params: EvolutionParams, bands: np.ndarray, init, keep):
        p, wkeep = _native_params(params)
        p.model = N.LSE_MODEL_BANDS
        p.n_bands = bands.shape[0]
        h = C.c_void_p()
        fmt = N.LSE_IMAGE_F32 if bands.dtype == np.float32 else N.LSE_IMAGE_F64
        rc = N.lib.lse_run_create(C.byref(h), C.byref(p), bands.shape[1], bands.shape[2],
                                  bands.ctypes.data_as(C.c_void_p), fmt, C.byref(init))
        del keep, wkeep
        if rc == N.LSE_ERR_DEGENERATE_SEED:
            raise DegenerateSeedError(N.lib.lse_last_error().decode())
        N.check(rc)
        self.h = h
        self.shape = bands.shape[1:]
        self._finalizer = weakref.finalize(self, N.lib.lse_run_destroy, h)


class BandEvolutionRun(EvolutionRun):
    """EvolutionRun (engine.py:193-269) over a (K, H, W) multi-band image."""

    def __init__(self, bands, seeds: SeedSpec, params: EvolutionParams, trace: bool = False):
        if params.model is not ModelKind.REGION:
            raise NotImplementedError("multi-band images run the region model")
        self.image = as_bands(bands)
        self.params = params
        self._reg_kernel = gaussian_kernel(params.sigma2, params.ts_reg)
        if isinstance(seeds, SeedSpec):
            self.seeds = seeds
            init, keep = _phi0_polygons(seeds)
        else:
            # an injected +-1 initial state (EvolutionState(phi=s * signs) with
            # reinit_period = 1 evolves identically for any s > 0)
            signs = np.ascontiguousarray(np.asarray(seeds), dtype=np.int8)
            if signs.shape != self.image.shape[1:] or not np.isin(signs, (-1, 1)).all():
                raise ValueError("initial signs must be a (H, W) array of +-1")
            self.seeds = SeedSpec(polygons=(np.zeros((3, 2)),), inside_sign=1)
            init = N.LsePhi0()
            init.kind = N.LSE_PHI0_SIGNS
            init.signs = signs.ctypes.data_as(C.POINTER(C.c_byte))
            init.scale = 1.0
            keep = signs
        self._dev = _BandDeviceRun(params, self.image, init, keep)
        self._version = 0
        self._snapshots = weakref.WeakSet()
        self.wall_time = 0.0
        self.trace = [(0, self._dev.contours())] if trace else None

    def band_stats(self) -> dict:
        """Peak passes reused because the partition moved no pixel (the
        means, D and max|D| are then bit-identical; LSE_BAND_REUSE=0 at
        creation recomputes them every iteration)."""
        out = (C.c_longlong * 2)()
        N.check(N.lib.lse_run_band_stats(self._dev.h, out))
        return dict(reused=int(out[0]), enabled=bool(out[1]))


def run_bands(bands, seeds: SeedSpec, params: EvolutionParams):
    """`run` (engine.py:272-277) for a multi-band image."""
    r = BandEvolutionRun(bands, seeds, params)
    r.advance(params.max_iters)
    return r.result()
