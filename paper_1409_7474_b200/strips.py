"""Row-strip decomposition of one evolution over several GPUs.

One process per GPU.  A rank owns a contiguous range of word-rows (32 image
rows each, the unit of the bit-packed state) of the global grid and keeps a
copy of one neighbouring word-row on each side (its halo).  Per iteration of
``_advance_once`` (engine.py:148-174) the ranks run:

  1. ``update``     u = phi + dt * v and b^{n+1} = sign(u) on their rows;
  2. halo exchange  first / last owned word-row of b^{n+1} -> neighbours
                    (phi^{n+1} = G * b^{n+1} and |grad phi| reach r + 1 <= 5
                    rows, inside one 32-row word, engine.py:160-169);
  3. ``partition``  signs of phi^{n+1} on their rows -> one 64-byte partial
                    (change of sum(I) / count over {phi >= 0}, grid.py:102-118,
                    plus the checkpoint mismatch count, engine.py:228-236);
  4. allgather      the partials, in rank order;
  5. ``finalize``   c+, c-, the next coefficients and the convergence state,
                    computed identically on every rank from the same partials.

Region/zhang runs need the partial exchange every iteration, edge runs only on
checkpoint iterations.  All device work and the communicator calls are
enqueued on the run's own CUDA stream, so the host never waits inside the loop.

The phases are backend-neutral: :class:`DeviceStrip` drives the C ABI
(``lse_strip_*``), and the tests drive the same :class:`StripDriver` with a CPU
stand-in over ``gloo``.  :class:`DistComm` exchanges through
``torch.distributed`` (NCCL on GPUs); :class:`LocalComm` runs several strips in
one process (single-GPU validation of the decomposition).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

WORD_ROWS = 32


@dataclass(frozen=True)
class StripWindow:
    """Rows of one strip: global word-rows [wr0, wr1) are owned; the local
    image spans global rows [y_lo, y_hi) (owned rows + halos); local word-rows
    [own_lo, own_hi) are the owned ones."""

    wr0: int
    wr1: int
    y_lo: int
    y_hi: int
    own_lo: int
    own_hi: int
    height: int
    width: int

    @property
    def rows(self) -> int:
        return self.y_hi - self.y_lo

    @property
    def own_rows(self) -> tuple[int, int]:
        """Owned global image rows [y0, y1)."""
        return self.wr0 * WORD_ROWS, min(self.height, self.wr1 * WORD_ROWS)

    @property
    def has_up(self) -> bool:
        return self.own_lo > 0

    @property
    def has_down(self) -> bool:
        return self.wr1 * WORD_ROWS < self.height


def plan_strips(height: int, width: int, world: int) -> list[StripWindow]:
    """Split the word-rows of a (height, width) grid into `world` strips."""
    hr = (height + WORD_ROWS - 1) // WORD_ROWS
    if world < 1 or world > hr:
        raise ValueError(f"cannot split {hr} word-rows over {world} ranks")
    base, extra = divmod(hr, world)
    out, wr = [], 0
    for k in range(world):
        n = base + (1 if k < extra else 0)
        wr0, wr1 = wr, wr + n
        top = 1 if wr0 > 0 else 0
        bot = 1 if wr1 < hr else 0
        y_lo = (wr0 - top) * WORD_ROWS
        y_hi = min(height, (wr1 + bot) * WORD_ROWS)
        out.append(StripWindow(wr0, wr1, y_lo, y_hi, top, top + n, height, width))
        wr = wr1
    return out


# ----------------------------------------------------------------- partials
# A partial is 64 bytes: (a_hi, a_lo, b_hi, b_lo) float64, (n_a, n_b, mism,
# pad) int64 -- lse_device.cuh TilePartial.
PARTIAL_BYTES = 64


def partial_counts(raw: np.ndarray) -> tuple[int, int]:
    """(n_a, n_b) of one partial given as 64 raw bytes."""
    q = np.frombuffer(np.ascontiguousarray(raw, dtype=np.uint8).tobytes(), dtype=np.int64)
    return int(q[4]), int(q[5])


# ------------------------------------------------------------ communicators
class LocalComm:
    """All strips in this process (one GPU): exchanges are device copies."""

    def __init__(self, strips):
        self.strips = list(strips)

    def _sync(self):
        for s in self.strips:
            s.synchronize()

    def allreduce_range(self, ranges):
        r = np.array(ranges, dtype=np.float64)
        g = (float(r[:, 0].min()), float(r[:, 1].max()), float(r[:, 2].max()))
        return [g] * len(ranges)

    def exchange_halos(self):
        self._sync()
        st = self.strips
        for k in range(len(st) - 1):
            up, dn = st[k], st[k + 1]
            dn.row(0).copy_(up.row(up.win.own_hi - 1))
            up.row(up.win.own_hi).copy_(dn.row(dn.win.own_lo))
        self._sync()

    def allgather(self, parts):
        import torch
        self._sync()
        g = torch.cat([p.reshape(-1) for p in parts])
        self._sync()
        return [g] * len(parts)


class DistComm:
    """One strip per rank; exchanges through torch.distributed on the strip's
    stream (NCCL on GPUs, gloo in the CPU tests)."""

    def __init__(self, strip, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.strips = [strip]
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._gathered = None
        self._stage = None

    def _stream(self):
        return self.strips[0].stream_context()

    def allreduce_range(self, ranges):
        import torch
        (mn, mx, am), = ranges
        with self._stream():       # H2D, the reduction and D2H all on the strip's stream
            t = torch.tensor([-mn, mx, am], dtype=torch.float64,
                             device=self.strips[0].comm_device)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
            t = t.cpu()
        return [(-float(t[0]), float(t[1]), float(t[2]))]

    def exchange_halos(self):
        """Own first/last word-row -> the neighbours' halo rows.  The rows
        travel through communicator-owned staging buffers (two 4*W-byte
        copies per side), so the collective library only ever sees memory
        its own allocator owns."""
        import torch
        s = self.strips[0]
        d = self.dist
        peer = lambda r: r if self.group is None else d.get_global_rank(self.group, r)  # noqa: E731
        sides = []
        if s.win.has_up:
            sides.append((s.win.own_lo, 0, peer(self.rank - 1)))
        if s.win.has_down:
            sides.append((s.win.own_hi - 1, s.win.own_hi, peer(self.rank + 1)))
        if not sides:
            return
        with self._stream():
            if self._stage is None:
                r0 = s.row(s.win.own_lo)
                self._stage = [(torch.empty_like(r0), torch.empty_like(r0)) for _ in range(2)]
            ops = []
            for (src, dst, pr), (tx, rx) in zip(sides, self._stage):
                tx.copy_(s.row(src))
                ops.append(d.P2POp(d.isend, tx, pr, self.group))
                ops.append(d.P2POp(d.irecv, rx, pr, self.group))
            for w in d.batch_isend_irecv(ops):
                w.wait()
            for (src, dst, pr), (tx, rx) in zip(sides, self._stage):
                s.row(dst).copy_(rx)

    def allgather(self, parts):
        import torch
        (p,), s = parts, self.strips[0]
        if self._gathered is None:
            self._gathered = torch.empty(self.world * p.numel(), dtype=p.dtype, device=p.device)
        with self._stream():
            self.dist.all_gather_into_tensor(self._gathered, p.reshape(-1), group=self.group)
        return [self._gathered]


# ------------------------------------------------------------------- driver
class StripDriver:
    """Runs the phases of the local strips in lock step with the other ranks."""

    def __init__(self, strips, comm, fused=None):
        self.strips = list(strips)
        self.comm = comm
        self.iteration = 0
        # one-pass iterations when every strip runs them (the same on every
        # rank: the strips' geometry decides; fused=False forces two passes)
        ok = all(getattr(s, "supports_fused", False) for s in self.strips)
        self.fused = ok if fused is None else (bool(fused) and ok)
        self._owed = False

    def setup(self):
        """Global image range, initial partition sums, seed-count check."""
        self.share_image_range()
        self.initialize()

    def share_image_range(self):
        """min / max / max|I| of the whole image on every rank (once per image)."""
        ranges = self.comm.allreduce_range([s.image_range() for s in self.strips])
        for s, g in zip(self.strips, ranges):
            s.set_image_range(g)

    def initialize(self):
        """Partition sums of the initial state, seed-count check (engine.py:202-216)."""
        self.iteration = 0
        self._owed = False
        parts = [s.prepare() for s in self.strips]
        gathered = self.comm.allgather(parts)
        for s in self.strips:
            s.synchronize()
        raw = gathered[0].cpu().numpy().view(np.uint8).reshape(-1, PARTIAL_BYTES)
        n_pos = sum(partial_counts(q)[0] for q in raw)     # pixels with b = +1
        w = self.strips[0].win
        n_total = w.height * w.width
        inside = n_pos if self.strips[0].inside_positive else n_total - n_pos
        if inside == 0 or inside == n_total:                # grid.py:88-93
            from .grid import DegenerateSeedError
            raise DegenerateSeedError("seed polygons cover no pixel centers" if inside == 0
                                      else "seed polygons cover the entire grid")
        for s, g in zip(self.strips, gathered):
            s.finalize(g, absolute=True)

    def step(self):
        if self.fused and self._owed:
            # partition of b^n + speculative update -> exchange partials ->
            # check / fix / redo -> halo rows of the final b^{n+1}
            parts = [s.fused() for s in self.strips]
            for s, g in zip(self.strips, self.comm.allgather(parts)):
                s.finalize(g, absolute=False)
            self.comm.exchange_halos()
            self.iteration += 1
            return
        need = [s.update() for s in self.strips]
        self.comm.exchange_halos()
        if need[0] and self.fused:
            self._owed = True           # taken by the next fused pass or flush()
        elif need[0]:
            self._partition()
        self.iteration += 1

    def _partition(self):
        parts = [s.partition() for s in self.strips]
        for s, g in zip(self.strips, self.comm.allgather(parts)):
            s.finalize(g, absolute=False)

    def flush(self):
        """The partition owed by the last update (convergence bookkeeping and
        the coefficients of the next iteration)."""
        if self._owed:
            self._partition()
            self._owed = False

    def advance(self, n):
        for _ in range(int(n)):
            self.step()
        self.flush()
        return [s.sync() for s in self.strips]


# ------------------------------------------------------------- device strip
class _CudaArray:
    """__cuda_array_interface__ view of device memory owned by a native run."""

    def __init__(self, ptr, n, typestr="<i4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None}


class DeviceStrip:
    """One rank's strip on its GPU, through the C ABI (lse_strip_*)."""

    def __init__(self, image_rows, win: StripWindow, seeds, params):
        import torch
        from . import _native as N
        from .engine import _native_params, _require_device_model
        from .grid import _poly_buffers

        _require_device_model(params.model)
        self.N, self.torch, self.win = N, torch, win
        img = np.ascontiguousarray(image_rows)
        if img.dtype not in (np.float32, np.float64):
            img = img.astype(np.float64)
        if img.shape != (win.rows, win.width):
            raise ValueError(f"strip image must be {(win.rows, win.width)}, got {img.shape}")
        p, wkeep = _native_params(params)
        xy, counts = _poly_buffers(seeds)
        init = N.LsePhi0()
        init.kind = N.LSE_PHI0_POLYGONS
        init.poly_xy = N.dptr(xy)
        init.poly_counts = counts.ctypes.data_as(N._llp)
        init.n_polys = len(counts)
        init.inside_sign = int(seeds.inside_sign)
        init.row_offset = win.y_lo
        self.inside_positive = int(seeds.inside_sign) > 0
        self._init, self._init_keep = init, (xy, counts)
        h = C.c_void_p()
        N.check(N.lib.lse_strip_create(C.byref(h), C.byref(p), win.rows, win.width,
                                       img.ctypes.data_as(C.c_void_p),
                                       1 if img.dtype == np.float32 else 0, C.byref(init),
                                       win.own_lo, win.own_hi, win.height * win.width))
        del wkeep
        self.h = h
        self._fin = weakref.finalize(self, N.lib.lse_run_destroy, h)
        hr, pw = C.c_int(), C.c_int()
        N.check(N.lib.lse_run_geometry(h, C.byref(hr), C.byref(pw)))
        self.pitch_words = pw.value
        dev = torch.cuda.current_device()
        self.comm_device = torch.device("cuda", dev)
        self.stream = torch.cuda.ExternalStream(N.lib.lse_run_stream(h), device=self.comm_device)
        self._part = torch.zeros(PARTIAL_BYTES, dtype=torch.uint8, device=self.comm_device)

    def reset(self):
        """Back to the seeded initial state (iteration 0); follow with
        StripDriver.initialize()."""
        self.N.check(self.N.lib.lse_run_set_state(self.h, C.byref(self._init)))

    def load_image(self, image_rows_ptr, is_f32=True):
        """Replace the strip's image rows from a host pointer (same shape)."""
        self.N.check(self.N.lib.lse_run_load_image(self.h, C.c_void_p(image_rows_ptr),
                                                   1 if is_f32 else 0))

    # -- phases ------------------------------------------------------------
    def stream_context(self):
        return self.torch.cuda.stream(self.stream)

    def synchronize(self):
        self.torch.cuda.synchronize(self.comm_device)

    def row(self, local_word_row):
        ptr = self.N.lib.lse_run_bits_row(self.h, int(local_word_row))
        if not ptr:
            raise IndexError(local_word_row)
        return self.torch.as_tensor(_CudaArray(ptr, self.pitch_words), device=self.comm_device)

    def image_range(self):
        out = np.empty(3)
        self.N.check(self.N.lib.lse_strip_image_range(self.h, self.N.dptr(out)))
        return tuple(float(v) for v in out)

    def set_image_range(self, g):
        arr = np.array(g, dtype=np.float64)
        self.N.check(self.N.lib.lse_strip_set_image_range(self.h, self.N.dptr(arr)))

    def prepare(self):
        self.N.check(self.N.lib.lse_strip_prepare(self.h, C.c_void_p(self._part.data_ptr())))
        return self._part

    def update(self):
        flag = C.c_int()
        self.N.check(self.N.lib.lse_strip_update(self.h, C.byref(flag)))
        return bool(flag.value)

    def partition(self):
        self.N.check(self.N.lib.lse_strip_partition(self.h, C.c_void_p(self._part.data_ptr())))
        return self._part

    @property
    def supports_fused(self):
        out = (C.c_longlong * 4)()
        self.N.check(self.N.lib.lse_run_spec_stats(self.h, out))
        return bool(out[3])

    def fused(self):
        """One-pass iteration: the owed partition + the next (speculative)
        update; returns this rank's partition partial."""
        self.N.check(self.N.lib.lse_strip_fused(self.h, C.c_void_p(self._part.data_ptr())))
        return self._part

    def finalize(self, gathered, absolute):
        n = gathered.numel() // PARTIAL_BYTES
        self.N.check(self.N.lib.lse_strip_finalize(self.h, C.c_void_p(gathered.data_ptr()), n,
                                                   1 if absolute else 0))

    def sync(self):
        st = self.N.LseStatus()
        self.N.check(self.N.lib.lse_strip_sync(self.h, C.byref(st)))
        return st

    # -- results -----------------------------------------------------------
    def own_mask(self, inside_sign):
        """mask() (engine.py:256-259) of the owned rows, uint8 0/1."""
        out = np.empty((self.win.rows, self.win.width), dtype=np.uint8)
        self.N.check(self.N.lib.lse_run_read_mask(
            self.h, out.ctypes.data_as(C.POINTER(C.c_ubyte)), int(inside_sign), 0))
        y0, y1 = self.win.own_rows
        return out[y0 - self.win.y_lo:y1 - self.win.y_lo]

    def own_phi(self):
        out = np.empty((self.win.rows, self.win.width), dtype=np.float64)
        self.N.check(self.N.lib.lse_run_read_phi(self.h, self.N.dptr(out)))
        y0, y1 = self.win.own_rows
        return out[y0 - self.win.y_lo:y1 - self.win.y_lo]


def strip_rows(image, win: StripWindow):
    """The rows of a full image that a strip holds (owned + halos)."""
    return np.ascontiguousarray(image[win.y_lo:win.y_hi])


def run_local_strips(image, seeds, params, n_strips, iters):
    """Single-process emulation: `n_strips` strips on the current GPU, driven
    exactly as the ranks of a multi-GPU run are (tests / validation)."""
    wins = plan_strips(image.shape[0], image.shape[1], n_strips)
    strips = [DeviceStrip(strip_rows(image, w), w, seeds, params) for w in wins]
    drv = StripDriver(strips, LocalComm(strips))
    drv.setup()
    status = drv.advance(iters)
    return drv, strips, status

