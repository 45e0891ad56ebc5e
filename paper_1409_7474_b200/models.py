"""Velocity fields (drop-in for lsekit/models.py).

The two fast evolutions of the paper run on the device: the edge-based
E_Td (Eq. 14; speed g * |grad phi|) and the region-based R_Td (Eq. 17;
max-normalized two-mean contrast times |grad phi|), plus the two baselines:
the mean-separation `zhang_velocity`, which shares the region kernels (only
the finalize coefficients differ), and the curvature-regularized
`cv_velocity`, which runs on the fp64 field path.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .kernels import gaussian_kernel

#: Gradient scale inside the edge function (models.py:20-26).
DEFAULT_EDGE_GAIN = 255.0


class ModelKind(enum.Enum):
    EDGE = "edge"
    REGION = "region"
    CHAN_VESE = "cv"
    ZHANG = "zhang"

    @classmethod
    def from_name(cls, name: str) -> "ModelKind":
        for kind in cls:
            if kind.value == name:
                return kind
        raise ValueError(f"unknown model {name!r}; expected one of "
                         f"{[k.value for k in cls]}")


@dataclass(frozen=True)
class ModelParams:
    """models.py:44-68 -- per-model free parameters, same validation."""

    sigma1: float = 1.0
    ts_pre: int = 9
    mu: float = 0.1
    nu: float = 1.0
    edge_gain: float = DEFAULT_EDGE_GAIN

    def __post_init__(self):
        if self.sigma1 <= 0:
            raise ValueError("sigma1 must be positive")
        if self.ts_pre < 1 or self.ts_pre % 2 == 0:
            raise ValueError("ts_pre must be an odd number >= 1")
        if self.mu < 0:
            raise ValueError("mu must be non-negative")
        if self.edge_gain <= 0:
            raise ValueError("edge_gain must be positive")


def edge_function(image: np.ndarray, sigma1: float, ts_pre: int,
                  gain: float = DEFAULT_EDGE_GAIN) -> np.ndarray:
    """models.py:71-81: 1 / (1 + |gain grad(G_sigma1 * I)|^2) (device)."""
    img = N.f64(image)
    if img.ndim != 2:
        raise ValueError("expected a 2-D field")
    w = N.f64(gaussian_kernel(sigma1, ts_pre).axis_weights)
    out = np.empty_like(img)
    N.check(N.lib.lse_edge_function(N.dptr(img), img.shape[0], img.shape[1], N.dptr(w), len(w),
                                    float(gain), N.dptr(out)))
    return out


def edge_velocity(g: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """models.py:84-90: g * |grad phi| (device)."""
    g = N.f64(g)
    phi = N.f64(phi)
    if g.shape != phi.shape:
        raise ValueError(f"shape mismatch: g {g.shape} vs phi {phi.shape}")
    if phi.ndim != 2 or phi.shape[0] < 2 or phi.shape[1] < 2:
        raise ValueError("gradient needs at least a 2x2 field")
    out = np.empty_like(phi)
    N.check(N.lib.lse_edge_velocity(N.dptr(g), N.dptr(phi), phi.shape[0], phi.shape[1],
                                    N.dptr(out)))
    return out


def region_velocity(image: np.ndarray, phi: np.ndarray) -> tuple[np.ndarray, bool]:
    """models.py:101-119: (D / max|D|) |grad phi|, D = (c+ - c-)(2I - c+ - c-).

    Degenerate partitions / zero contrast give (zeros, True) (device).
    """
    image = N.f64(image)
    phi = N.f64(phi)
    if image.shape != phi.shape:
        raise ValueError(f"shape mismatch: image {image.shape} vs phi {phi.shape}")
    if phi.ndim != 2:
        raise ValueError("expected a 2-D field")
    out = np.empty_like(phi)
    deg = N.C.c_int(0)
    N.check(N.lib.lse_region_velocity(N.dptr(image), N.dptr(phi), phi.shape[0], phi.shape[1],
                                      N.dptr(out), N.C.byref(deg)))
    return out, bool(deg.value)


def cv_velocity(image, phi, mu, eps_guard=1e-10):
    """models.py:122-141: [(c+ - c-)(2I - c+ - c-) + mu * kappa] * |grad phi|,
    un-normalized; the data term is zero when a side is empty (device)."""
    image = N.f64(image)
    phi = N.f64(phi)
    if image.shape != phi.shape:
        raise ValueError("image and phi shapes differ")
    if eps_guard != 1e-10 and mu != 0.0:
        from .kernels import curvature, gradient_magnitude
        from .grid import region_means, DegeneratePartitionError
        try:
            c_plus, c_minus = region_means(image, phi)
            data = (c_plus - c_minus) * (2.0 * image - c_plus - c_minus)
        except DegeneratePartitionError:
            data = np.zeros_like(phi)
        return (data + mu * curvature(phi, eps_guard)) * gradient_magnitude(phi)
    out = np.empty_like(phi)
    N.check(N.lib.lse_cv_velocity(N.dptr(image), N.dptr(phi), phi.shape[0], phi.shape[1],
                                  float(mu), N.dptr(out)))
    return out


def zhang_velocity(image, phi, nu):
    """models.py:144-162: nu * (I - m) / max|I - m| * |grad phi|, m = (c+ + c-)/2.

    Degenerate partitions / constant images give (zeros, True) (device).
    """
    image = N.f64(image)
    phi = N.f64(phi)
    if image.shape != phi.shape:
        raise ValueError(f"shape mismatch: image {image.shape} vs phi {phi.shape}")
    if phi.ndim != 2:
        raise ValueError("expected a 2-D field")
    out = np.empty_like(phi)
    deg = N.C.c_int(0)
    N.check(N.lib.lse_zhang_velocity(N.dptr(image), N.dptr(phi), phi.shape[0], phi.shape[1],
                                     float(nu), N.dptr(out), N.C.byref(deg)))
    return out, bool(deg.value)
