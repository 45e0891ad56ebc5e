"""The evolution loop (drop-in for lsekit/engine.py), driven on the device.

Same parameters, validation, warnings, state/result types, error messages
and resumability as the reference (engine.py:1-294).  `EvolutionRun` owns a
device run handle (liblse_b200.so): the image, the binary level-set state,
the partition sums and the checkpoint history live in HBM; `advance(n)`
launches the fused kernels and returns after the device finished.  The
float64 phi of `state` is materialized lazily (bit-identical to the
reference's G * b), so polling `run.state.iteration` costs no transfer.
"""

from __future__ import annotations

import ctypes as C
import time
import warnings
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .grid import SeedSpec, as_field, as_image, rasterize_seeds, _poly_buffers
from .kernels import Kernel2D, gaussian_kernel
from .models import ModelKind, ModelParams

#: Time steps above this empirically destabilize the explicit update (engine.py:26).
DT_STABILITY_LIMIT = 25.0


class NumericalInstabilityError(RuntimeError):
    """Raised when the update produces NaN/Inf; names the iteration (engine.py:29-37)."""

    def __init__(self, iteration: int):
        super().__init__(
            f"numerical instability: non-finite level-set values at "
            f"iteration {iteration} (time steps above {DT_STABILITY_LIMIT:g} "
            f"are prone to this)")
        self.iteration = iteration


@dataclass(frozen=True)
class EvolutionParams:
    """Knobs of the evolution loop (engine.py:40-81), identical validation."""

    model: ModelKind
    dt: float = 15.0
    sigma2: float = 1.0
    ts_reg: int = 9
    reinit_period: int = 1
    reg_period: int = 1
    max_iters: int = 1000
    conv_check_every: int = 10
    conv_window: int = 3
    model_params: ModelParams = field(default_factory=ModelParams)

    def __post_init__(self):
        if self.dt <= 0:
            raise ValueError("dt must be positive")
        if self.sigma2 <= 0:
            raise ValueError("sigma2 must be positive")
        if self.ts_reg < 1 or self.ts_reg % 2 == 0:
            raise ValueError("ts_reg must be an odd number >= 1")
        if self.reinit_period < 0:
            raise ValueError("reinit_period must be >= 0 (0 = never)")
        if self.reg_period < 1:
            raise ValueError("reg_period must be >= 1")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.conv_check_every < 1 or self.conv_window < 1:
            raise ValueError("convergence cadence values must be >= 1")
        if self.model is ModelKind.EDGE and self.reinit_period < 1:
            raise ValueError("the edge model requires reinit_period >= 1")
        if self.dt > DT_STABILITY_LIMIT:
            warnings.warn(
                f"dt={self.dt:g} exceeds {DT_STABILITY_LIMIT:g}; unstable "
                f"results may arise", RuntimeWarning, stacklevel=2)


def default_params(model: ModelKind, **overrides) -> EvolutionParams:
    """engine.py:84-95: recommended defaults per model."""
    base = dict(model=model, dt=15.0, sigma2=1.0, ts_reg=9,
                reinit_period=1, reg_period=1)
    if model is ModelKind.CHAN_VESE:
        base.update(dt=0.8, reinit_period=20)
    mp_fields = {k: overrides.pop(k) for k in
                 ("sigma1", "ts_pre", "mu", "nu", "edge_gain")
                 if k in overrides}
    base.update(overrides)
    return EvolutionParams(model_params=ModelParams(**mp_fields), **base)


@dataclass(frozen=True)
class EvolutionState:
    phi: np.ndarray
    iteration: int = 0
    converged: bool = False
    degenerate: bool = False


@dataclass(frozen=True)
class ExtractionResult:
    """engine.py:106-120."""

    mask: np.ndarray
    object_sign: int
    iterations: int
    wall_time: float
    converged: bool
    degenerate: bool
    trace: tuple | None = None


class _DeviceState(EvolutionState):
    """An EvolutionState snapshot whose phi still lives on the device.

    phi is downloaded on first access; if the run moves on first, the
    owning run downloads it before changing the device state, so the
    snapshot keeps the semantics of the reference's immutable arrays.
    """

    __hash__ = object.__hash__

    def __init__(self, phi=None, iteration=0, converged=False, degenerate=False, *,
                 _run=None, _version=None):
        object.__setattr__(self, "iteration", iteration)
        object.__setattr__(self, "converged", converged)
        object.__setattr__(self, "degenerate", degenerate)
        object.__setattr__(self, "_run", _run)
        object.__setattr__(self, "_version", _version)
        object.__setattr__(self, "_phi", phi)

    @property
    def phi(self):
        if self._phi is None:
            object.__setattr__(self, "_phi", self._run._read_phi())
        return self._phi

    def _detach(self):
        if self._phi is None:
            self.phi  # noqa: B018  (materialize)


def _require_device_model(model: ModelKind):
    if model not in (ModelKind.REGION, ModelKind.EDGE, ModelKind.ZHANG, ModelKind.CHAN_VESE):
        raise NotImplementedError(f"unknown model {model!r}")


def _native_params(params: EvolutionParams, max_iters=None, conv_check_every=None):
    mp = params.model_params
    wreg = np.ascontiguousarray(gaussian_kernel(params.sigma2, params.ts_reg).axis_weights)
    wpre = np.ascontiguousarray(gaussian_kernel(mp.sigma1, mp.ts_pre).axis_weights)
    p = N.LseParams()
    p.model = {ModelKind.REGION: N.LSE_MODEL_REGION, ModelKind.ZHANG: N.LSE_MODEL_ZHANG,
               ModelKind.EDGE: N.LSE_MODEL_EDGE, ModelKind.CHAN_VESE: N.LSE_MODEL_CV}[params.model]
    p.dt = float(params.dt)
    p.sigma2 = float(params.sigma2)
    p.ts_reg = int(params.ts_reg)
    p.reinit_period = int(params.reinit_period)
    p.reg_period = int(params.reg_period)
    p.max_iters = int(params.max_iters if max_iters is None else max_iters)
    p.conv_check_every = int(params.conv_check_every if conv_check_every is None
                             else conv_check_every)
    p.conv_window = int(params.conv_window)
    p.sigma1 = float(mp.sigma1)
    p.ts_pre = int(mp.ts_pre)
    p.edge_gain = float(mp.edge_gain)
    p.reg_weights = N.dptr(wreg)
    p.pre_weights = N.dptr(wpre)
    p.nu = float(mp.nu)
    p.mu = float(mp.mu)
    return p, (wreg, wpre)


def _phi0_polygons(seeds: SeedSpec):
    xy, counts = _poly_buffers(seeds)
    s = N.LsePhi0()
    s.kind = N.LSE_PHI0_POLYGONS
    s.poly_xy = N.dptr(xy)
    s.poly_counts = counts.ctypes.data_as(N._llp)
    s.n_polys = len(counts)
    s.inside_sign = int(seeds.inside_sign)
    return s, (xy, counts)


def _phi0_field(phi, iteration=0, converged=False, degenerate=False):
    f = N.f64(phi)
    s = N.LsePhi0()
    s.kind = N.LSE_PHI0_FIELD
    s.field = N.dptr(f)
    s.iteration = int(iteration)
    s.converged = int(bool(converged))
    s.degenerate = int(bool(degenerate))
    return s, f


class _DeviceRun:
    """Owner of one native run handle (released on garbage collection)."""

    def __init__(self, params: EvolutionParams, image: np.ndarray, init, keep,
                 max_iters=None, conv_check_every=None):
        p, wkeep = _native_params(params, max_iters, conv_check_every)
        h = C.c_void_p()
        if image.dtype == np.uint8 and image.ndim == 3 and image.shape[2] == 3:
            fmt = N.LSE_IMAGE_RGB8       # decoded to the loader's luma on the device
        else:
            fmt = N.LSE_IMAGE_F32 if image.dtype == np.float32 else N.LSE_IMAGE_F64
        rc = N.lib.lse_run_create(C.byref(h), C.byref(p), image.shape[0], image.shape[1],
                                  image.ctypes.data_as(C.c_void_p), fmt, C.byref(init))
        del keep, wkeep
        if rc == N.LSE_ERR_DEGENERATE_SEED:
            from .grid import DegenerateSeedError
            raise DegenerateSeedError(N.lib.lse_last_error().decode())
        if rc == N.LSE_ERR_ARG and b"non-finite" in N.lib.lse_last_error():
            raise ValueError("grid contains non-finite values")
        N.check(rc)
        self.h = h
        self.shape = image.shape[:2]
        self._finalizer = weakref.finalize(self, N.lib.lse_run_destroy, h)

    def advance(self, n):
        st = N.LseStatus()
        rc = N.lib.lse_run_advance(self.h, int(n), C.byref(st))
        if rc == N.LSE_ERR_INSTABILITY:
            raise NumericalInstabilityError(int(st.instability_iteration))
        N.check(rc)
        return st

    def status(self):
        st = N.LseStatus()
        N.check(N.lib.lse_run_status(self.h, C.byref(st)))
        return st

    def read_phi(self):
        out = np.empty(self.shape, dtype=np.float64)
        N.check(N.lib.lse_run_read_phi(self.h, N.dptr(out)))
        return out

    def read_mask(self, inside_sign):
        out = np.empty(self.shape, dtype=np.uint8)
        N.check(N.lib.lse_run_read_mask(self.h, out.ctypes.data_as(C.POINTER(C.c_ubyte)),
                                        int(inside_sign), 0))
        return out.view(bool)

    def contours(self):
        """Zero-level contours of the current phi, computed on the device."""
        c = C.c_void_p()
        N.check(N.lib.lse_run_contours(self.h, C.byref(c)))
        return N.take_contours(c)

    def set_state(self, st: EvolutionState):
        s, keep = _phi0_field(st.phi, st.iteration, st.converged, st.degenerate)
        N.check(N.lib.lse_run_set_state(self.h, C.byref(s)))
        del keep


def init_state(image: np.ndarray, seeds: SeedSpec,
               params: EvolutionParams) -> EvolutionState:
    """engine.py:123-133: rasterize the seeds into the binary initial field."""
    image = as_field(image)
    h, w = image.shape
    phi0 = rasterize_seeds(seeds, w, h)
    if params.model is ModelKind.CHAN_VESE:             # engine.py:129-132
        from .kernels import signed_distance
        sd = signed_distance(phi0 == seeds.inside_sign)
        phi0 = sd if seeds.inside_sign < 0 else -sd
    return EvolutionState(phi=phi0, iteration=0)


def step(state: EvolutionState, image: np.ndarray,
         params: EvolutionParams) -> EvolutionState:
    """engine.py:177-190: one stateless iteration (edge indicator rebuilt per call)."""
    if state.converged:
        raise ValueError("evolution already converged")
    _require_device_model(params.model)
    image = as_image(np.asarray(image, dtype=np.float64))
    init, keep = _phi0_field(state.phi, state.iteration, False, state.degenerate)
    run = _DeviceRun(params, image, init, keep, max_iters=int(state.iteration) + 1,
                     conv_check_every=1 << 62)
    st = run.advance(1)
    return EvolutionState(phi=run.read_phi(), iteration=int(st.iteration),
                          degenerate=bool(state.degenerate or st.degenerate))


class EvolutionRun:
    """Resumable driver (engine.py:193-269).

    ``advance(n)`` performs at most n iterations on the device, stopping
    early at convergence or max_iters; calling it repeatedly walks the exact
    same trajectory a single run() would.
    """

    def __init__(self, image: np.ndarray, seeds: SeedSpec,
                 params: EvolutionParams, trace: bool = False):
        _require_device_model(params.model)
        # two-mean models: the device's image statistics pass rejects
        # non-finite values (as_field's ValueError, grid.py:24-31)
        self.image = as_image(image, check_finite=params.model not in (ModelKind.REGION,
                                                                        ModelKind.ZHANG))
        self.seeds = seeds
        self.params = params
        self._reg_kernel = gaussian_kernel(params.sigma2, params.ts_reg)
        init, keep = _phi0_polygons(seeds)
        self._dev = _DeviceRun(params, self.image, init, keep)
        self._version = 0
        self._snapshots = weakref.WeakSet()
        self.wall_time = 0.0
        self.trace = None
        if trace:                                       # engine.py:214-216
            self.trace = [(0, self._dev.contours())]

    # -- state -----------------------------------------------------------
    def _read_phi(self):
        return self._dev.read_phi()

    def _before_mutation(self):
        for snap in list(self._snapshots):
            if snap._version == self._version:
                snap._detach()
        self._version += 1

    @property
    def state(self) -> EvolutionState:
        st = self._dev.status()
        snap = _DeviceState(iteration=int(st.iteration), converged=bool(st.converged),
                            degenerate=bool(st.degenerate), _run=self, _version=self._version)
        self._snapshots.add(snap)
        return snap

    @state.setter
    def state(self, st: EvolutionState):
        if isinstance(st, _DeviceState) and st._run is self and st._version == self._version:
            return
        self._before_mutation()
        self._dev.set_state(st)

    @property
    def converged(self) -> bool:
        return bool(self._dev.status().converged)

    def advance(self, n_steps: int) -> EvolutionState:
        """engine.py:242-254: run up to n_steps iterations."""
        if n_steps < 0:
            raise ValueError("n_steps must be >= 0")
        self._before_mutation()
        t0 = time.perf_counter()
        try:
            if self.trace is None:
                self._dev.advance(n_steps)
            else:
                self._advance_traced(int(n_steps))
        finally:
            self.wall_time += time.perf_counter() - t0
        return self.state

    def _advance_traced(self, n_steps):
        """Checkpoint to checkpoint, appending the contours of phi at every
        checkpoint iteration (engine.py:226-238); the device trajectory is the
        same as one advance(n_steps)."""
        cce = self.params.conv_check_every
        left = n_steps
        while left > 0:
            st0 = self._dev.status()
            if st0.converged or st0.iteration >= self.params.max_iters:
                break
            k = min(left, cce - int(st0.iteration) % cce)
            st = self._dev.advance(k)
            done = int(st.iteration) - int(st0.iteration)
            left -= done
            if done > 0 and int(st.iteration) % cce == 0:
                self.trace.append((int(st.iteration), self._dev.contours()))
            if done < k:
                break

    def mask(self) -> np.ndarray:
        """engine.py:256-259: the binary class carrying the seed sign."""
        return self._dev.read_mask(self.seeds.inside_sign)

    def contours(self):
        """engine.py:260-261, on the device state (no phi download)."""
        return self._dev.contours()

    def result(self) -> ExtractionResult:
        st = self._dev.status()
        return ExtractionResult(
            mask=self.mask(), object_sign=self.seeds.inside_sign,
            iterations=int(st.iteration), wall_time=self.wall_time,
            converged=bool(st.converged), degenerate=bool(st.degenerate),
            trace=tuple(self.trace) if self.trace is not None else None)

    def set_native_option(self, name: str, value: int) -> None:
        """Tune the device run (e.g. "skip_uniform" 0/1); results are unchanged."""
        N.check(N.lib.lse_run_set_option(self._dev.h, name.encode(), int(value)))

    def fallback_count(self) -> int:
        """fp64 re-evaluations of near-tie pixels so far (diagnostics)."""
        return int(self._dev.status().exact_fallbacks)

    def spec_stats(self) -> dict:
        """Speculative fused iterations of this run (diagnostics; results are
        the same with LSE_FUSED=0): launched, redone whole, fix-list pixels."""
        out = (C.c_longlong * 4)()
        N.check(N.lib.lse_run_spec_stats(self._dev.h, out))
        return dict(fused=int(out[0]), redos=int(out[1]), fixes=int(out[2]),
                    enabled=bool(out[3]))

    def resident_stats(self) -> dict:
        """Resident-kernel path of small images (diagnostics; results are the
        same with LSE_RESIDENT=0): enabled, barrier kind, CTAs, calls served."""
        out = (C.c_longlong * 5)()
        N.check(N.lib.lse_run_resident_stats(self._dev.h, out))
        return dict(enabled=bool(out[0]), grid=bool(out[1]), ctas=int(out[2]), calls=int(out[3]),
                    tasks_per_warp=int(out[4]))

    def path_counts(self) -> tuple[int, int]:
        st = self._dev.status()
        return int(st.fast_iterations), int(st.generic_iterations)


def run(image: np.ndarray, seeds: SeedSpec, params: EvolutionParams,
        trace: bool = False) -> ExtractionResult:
    """engine.py:272-277: evolve to convergence (or max_iters)."""
    r = EvolutionRun(image, seeds, params, trace=trace)
    r.advance(params.max_iters)
    return r.result()


def extract_contours(phi: np.ndarray):
    """engine.py:280-294: zero-level polylines of phi as (x, y) arrays.

    Marching squares runs on the device (lse_contours_from_field; the
    published scikit-image find_contours algorithm the reference calls,
    level 0, low values fully connected); a single-signed field yields []."""
    phi = np.ascontiguousarray(phi, dtype=np.float64)
    if not ((phi > 0).any() and (phi < 0).any()):
        return []
    if phi.ndim != 2:
        raise ValueError("Only 2D arrays are supported.")
    c = C.c_void_p()
    N.check(N.lib.lse_contours_from_field(phi.ctypes.data_as(C.c_void_p), 0, phi.shape[0],
                                          phi.shape[1], C.byref(c)))
    return N.take_contours(c)
