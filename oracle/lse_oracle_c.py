"""ctypes wrapper of oracle/lse_oracle.c -- TEST / BASELINE INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liblse_oracle.so")

_dp = C.POINTER(C.c_double)


class OracleParamsC(C.Structure):
    _fields_ = [("model", C.c_int), ("dt", C.c_double), ("ts_reg", C.c_int),
                ("reinit_period", C.c_int), ("reg_period", C.c_int), ("max_iters", C.c_longlong),
                ("conv_check_every", C.c_longlong), ("conv_window", C.c_longlong),
                ("edge_gain", C.c_double), ("ts_pre", C.c_int), ("reg_w", _dp), ("pre_w", _dp),
                ("nu", C.c_double), ("nbands", C.c_int)]


def load():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-C", HERE])
    lib = C.CDLL(LIB)
    lib.oracle_create.restype = C.c_void_p
    lib.oracle_create.argtypes = [_dp, C.c_int, C.c_int, C.POINTER(OracleParamsC), _dp]
    lib.oracle_destroy.restype = None
    lib.oracle_destroy.argtypes = [C.c_void_p]
    lib.oracle_advance.restype = C.c_longlong
    lib.oracle_advance.argtypes = [C.c_void_p, C.c_longlong]
    lib.oracle_state.restype = None
    lib.oracle_state.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_int),
                                 C.POINTER(C.c_int)]
    lib.oracle_edge_function.restype = None
    lib.oracle_edge_function.argtypes = [_dp, C.c_int, C.c_int, _dp, C.c_int, C.c_double, _dp]
    lib.oracle_threads.restype = C.c_int
    lib.oracle_set_threads.restype = None
    lib.oracle_set_threads.argtypes = [C.c_int]
    return lib


def set_threads(n):
    """OpenMP threads of the C restatement (1: the reference's single core)."""
    load().oracle_set_threads(int(n))


class COracleRun:
    """EvolutionRun restated in C; one advance() call = one fresh run segment."""

    def __init__(self, image, phi0, p, gaussian_weights):
        """image: (H, W), or (K, H, W) bands for the multi-band region term
        (p.model "region" with K planes runs model 3)."""
        self.lib = load()
        self.image = np.ascontiguousarray(image, dtype=np.float64)
        nb = self.image.shape[0] if self.image.ndim == 3 else 1
        self.phi = np.ascontiguousarray(phi0, dtype=np.float64).copy()
        self.wreg = np.ascontiguousarray(gaussian_weights(p.sigma2, p.ts_reg))
        self.wpre = np.ascontiguousarray(gaussian_weights(p.sigma1, p.ts_pre))
        model = {"edge": 0, "region": 1, "zhang": 2}[p.model]
        if self.image.ndim == 3:
            if model != 1:
                raise ValueError("multi-band images run the region model")
            model = 3
        self.cp = OracleParamsC(model, p.dt, p.ts_reg, p.reinit_period,
                                p.reg_period, p.max_iters, p.conv_check_every, p.conv_window,
                                p.edge_gain, p.ts_pre, self.wreg.ctypes.data_as(_dp),
                                self.wpre.ctypes.data_as(_dp), getattr(p, "nu", 1.0), nb)
        h, w = self.image.shape[-2:]
        self.ctx = self.lib.oracle_create(self.image.ctypes.data_as(_dp), h, w,
                                          C.byref(self.cp), self.phi.ctypes.data_as(_dp))
        self.iteration = 0
        self.converged = False
        self.degenerate = False

    def __del__(self):
        if getattr(self, "ctx", None):
            self.lib.oracle_destroy(self.ctx)
            self.ctx = None

    def advance(self, n):
        err = self.lib.oracle_advance(self.ctx, n)
        it, conv, deg = C.c_longlong(), C.c_int(), C.c_int()
        self.lib.oracle_state(self.ctx, C.byref(it), C.byref(conv), C.byref(deg))
        self.iteration, self.converged, self.degenerate = it.value, bool(conv.value), bool(deg.value)
        return int(err)

    def threads(self):
        return int(self.lib.oracle_threads())
