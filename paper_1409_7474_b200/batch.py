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


# ------------------------------------------------------- multi-GPU sharding
def shard(n_tiles: int, rank: int, world: int) -> list[int]:
    """Tiles of one rank: k = rank, rank + world, ... (the
    tiles are independent units, so a rank's share needs no data-path
    collective; the split is even to within one tile)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return list(range(rank, n_tiles, world))


def run_tiles_sharded(make_tile, n_tiles: int, rank: int | None = None,
                      world: int | None = None, gather: str = "all", runner=None):
    """`run` for n_tiles independent tiles spread over the ranks of the
    default torch.distributed group (one process per GPU).

    make_tile(k) -> (image, seeds, params) builds tile k; each rank runs its
    shard(n_tiles, rank, world) as one TileBatch on its own GPU (runner:
    list of (image, seeds, params) -> list of ExtractionResult, default
    run_tiles).  The only communication is the host-side gather of the
    per-tile results afterwards: gather = "all" (every rank gets all n_tiles
    results in tile order), "rank0" (rank 0 does, the others get None) or
    "none" (each rank returns {k: result} of its own tiles).
    """
    import torch.distributed as dist
    if rank is None or world is None:
        on = dist.is_available() and dist.is_initialized()
        rank = dist.get_rank() if on else 0
        world = dist.get_world_size() if on else 1
    mine = shard(n_tiles, rank, world)
    runner = runner or (lambda items: run_tiles([i[0] for i in items], [i[1] for i in items],
                                                [i[2] for i in items]))
    items = [make_tile(k) for k in mine]
    local = dict(zip(mine, runner(items) if items else []))
    if gather == "none" or world == 1:
        return local if gather == "none" else [local[k] for k in range(n_tiles)]
    parts = [None] * world
    if gather == "all":
        dist.all_gather_object(parts, local)
    else:
        dist.gather_object(local, parts if rank == 0 else None, dst=0)
        if rank != 0:
            return None
    merged = {}
    for p in parts:
        merged.update(p)
    if sorted(merged) != list(range(n_tiles)):
        raise RuntimeError("tile gather lost tiles")
    return [merged[k] for k in range(n_tiles)]
