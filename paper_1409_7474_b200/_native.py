"""ctypes binding of the C ABI in include/lse_b200.h (liblse_b200.so).

The library is built in-tree (`make` or `__graft_entry__.build()`).  There is
no fallback: a missing library raises ImportError at import time, and every
call that needs a device raises RuntimeError when none is visible.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSE_LIB_PATH") or os.path.join(_HERE, "_lib", "liblse_b200.so")

LSE_OK = 0
LSE_ERR_ARG = 1
LSE_ERR_CUDA = 2
LSE_ERR_INSTABILITY = 3
LSE_ERR_DEGENERATE = 4
LSE_ERR_NODEVICE = 5
LSE_ERR_DEGENERATE_SEED = 6
LSE_ERR_UNSUPPORTED = 7

LSE_MODEL_EDGE = 0
LSE_MODEL_REGION = 1
LSE_MODEL_ZHANG = 2
LSE_MODEL_BANDS = 3
LSE_MODEL_CV = 4
LSE_PARTIAL_BYTES = 64
LSE_IMAGE_F64, LSE_IMAGE_F32, LSE_IMAGE_RGB8 = 0, 1, 2

LSE_PHI0_FIELD = 0
LSE_PHI0_SIGNS = 1
LSE_PHI0_POLYGONS = 2

_dp = C.POINTER(C.c_double)
_llp = C.POINTER(C.c_longlong)


class LseParams(C.Structure):
    _fields_ = [("model", C.c_int), ("dt", C.c_double), ("sigma2", C.c_double),
                ("ts_reg", C.c_int), ("reinit_period", C.c_int), ("reg_period", C.c_int),
                ("max_iters", C.c_longlong), ("conv_check_every", C.c_longlong),
                ("conv_window", C.c_longlong), ("sigma1", C.c_double), ("ts_pre", C.c_int),
                ("edge_gain", C.c_double), ("reg_weights", _dp), ("pre_weights", _dp),
                ("nu", C.c_double), ("n_bands", C.c_int), ("mu", C.c_double)]


class LsePhi0(C.Structure):
    _fields_ = [("kind", C.c_int), ("field", _dp), ("signs", C.POINTER(C.c_byte)),
                ("scale", C.c_double), ("poly_xy", _dp), ("poly_counts", _llp),
                ("n_polys", C.c_longlong), ("inside_sign", C.c_int),
                ("iteration", C.c_longlong), ("converged", C.c_int), ("degenerate", C.c_int),
                ("row_offset", C.c_longlong)]


class LseStatus(C.Structure):
    _fields_ = [("iteration", C.c_longlong), ("converged", C.c_int), ("degenerate", C.c_int),
                ("instability_iteration", C.c_longlong), ("exact_fallbacks", C.c_longlong),
                ("fast_iterations", C.c_longlong), ("generic_iterations", C.c_longlong)]


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first (make, or "
        "python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")

lib = C.CDLL(LIB_PATH)

_vp = C.c_void_p
_i = C.c_int
_ll = C.c_longlong
_SIGS = {
    "lse_abi_version": (_i, []),
    "lse_last_error": (C.c_char_p, []),
    "lse_device_count": (_i, []),
    "lse_run_create": (_i, [C.POINTER(_vp), C.POINTER(LseParams), _ll, _ll, _vp, _i,
                            C.POINTER(LsePhi0)]),
    "lse_run_load_image": (_i, [_vp, _vp, _i]),
    "lse_run_set_state": (_i, [_vp, C.POINTER(LsePhi0)]),
    "lse_run_advance": (_i, [_vp, _ll, C.POINTER(LseStatus)]),
    "lse_run_status": (_i, [_vp, C.POINTER(LseStatus)]),
    "lse_run_read_phi": (_i, [_vp, _dp]),
    "lse_run_read_mask": (_i, [_vp, C.POINTER(C.c_ubyte), _i, _i]),
    "lse_run_begin_timing": (_i, [_vp]),
    "lse_run_end_timing": (_i, [_vp, _dp]),
    "lse_launch_count": (_ll, []),
    "lse_check_enabled": (_i, []),
    "lse_check_stats": (_i, [_dp, _i]),
    "lse_run_set_option": (_i, [_vp, C.c_char_p, _ll]),
    "lse_run_set_profiling": (_i, [_vp, _i]),
    "lse_run_kernel_times": (_i, [_vp, _dp, _llp, _dp, _llp]),
    "lse_run_spec_stats": (_i, [_vp, _llp]),
    "lse_run_band_stats": (_i, [_vp, _llp]),
    "lse_run_resident_stats": (_i, [_vp, _llp]),
    "lse_run_destroy": (None, [_vp]),
    "lse_batch_create": (_i, [C.POINTER(_vp), C.POINTER(_vp), _i]),
    "lse_batch_advance": (_i, [_vp, _ll, C.POINTER(LseStatus)]),
    "lse_batch_destroy": (None, [_vp]),
    "lse_batch_set_timing": (_i, [_vp, _i]),
    "lse_batch_elapsed": (_i, [_vp, _dp, _llp]),
    "lse_strip_create": (_i, [C.POINTER(_vp), C.POINTER(LseParams), _ll, _ll, _vp, _i,
                              C.POINTER(LsePhi0), _i, _i, _ll]),
    "lse_strip_image_range": (_i, [_vp, _dp]),
    "lse_strip_set_image_range": (_i, [_vp, _dp]),
    "lse_strip_prepare": (_i, [_vp, _vp]),
    "lse_strip_update": (_i, [_vp, C.POINTER(C.c_int)]),
    "lse_strip_partition": (_i, [_vp, _vp]),
    "lse_strip_finalize": (_i, [_vp, _vp, _i, _i]),
    "lse_strip_fused": (_i, [_vp, _vp]),
    "lse_strip_sync": (_i, [_vp, C.POINTER(LseStatus)]),
    "lse_run_stream": (_vp, [_vp]),
    "lse_run_bits_row": (_vp, [_vp, _i]),
    "lse_run_geometry": (_i, [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "lse_edge_function": (_i, [_dp, _ll, _ll, _dp, _i, C.c_double, _dp]),
    "lse_convolve_same": (_i, [_dp, _ll, _ll, _dp, _i, _dp]),
    "lse_correlate2d": (_i, [_dp, _ll, _ll, _dp, _i, _dp]),
    "lse_gradient": (_i, [_dp, _ll, _ll, _dp, _dp, _dp]),
    "lse_binarize": (_i, [_dp, _ll, _dp]),
    "lse_region_means": (_i, [_dp, _dp, _ll, _ll, _dp, _dp]),
    "lse_region_velocity": (_i, [_dp, _dp, _ll, _ll, _dp, C.POINTER(C.c_int)]),
    "lse_curvature": (_i, [_dp, _ll, _ll, C.c_double, _dp]),
    "lse_signed_distance": (_i, [C.POINTER(C.c_ubyte), _ll, _ll, _dp]),
    "lse_cv_velocity": (_i, [_dp, _dp, _ll, _ll, C.c_double, _dp]),
    "lse_zhang_velocity": (_i, [_dp, _dp, _ll, _ll, C.c_double, _dp, C.POINTER(C.c_int)]),
    "lse_edge_velocity": (_i, [_dp, _dp, _ll, _ll, _dp]),
    "lse_rasterize_seeds": (_i, [_dp, _llp, _ll, _i, _ll, _ll, C.POINTER(C.c_byte)]),
    "lse_contours_from_field": (_i, [_vp, _i, _ll, _ll, C.POINTER(_vp)]),
    "lse_run_contours": (_i, [_vp, C.POINTER(_vp)]),
    "lse_contours_size": (_i, [_vp, _llp, _llp]),
    "lse_contours_read": (_i, [_vp, _llp, _dp]),
    "lse_contours_destroy": (None, [_vp]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
_lock = threading.Lock()


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc):
    if rc != LSE_OK:
        msg = lib.lse_last_error().decode(errors="replace")
        raise NativeError(rc, msg or f"lse error {rc}")


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def take_contours(c) -> list:
    """Reads and frees an lse_contours handle: a list of (n, 2) float64 (x, y)
    arrays, as extract_contours returns them (engine.py:280-294)."""
    try:
        nc, npt = C.c_longlong(), C.c_longlong()
        check(lib.lse_contours_size(c, C.byref(nc), C.byref(npt)))
        off = np.empty(nc.value + 1, dtype=np.int64)
        xy = np.empty((max(npt.value, 1), 2), dtype=np.float64)
        check(lib.lse_contours_read(c, off.ctypes.data_as(_llp), dptr(xy)))
    finally:
        lib.lse_contours_destroy(c)
    return [xy[off[k]:off[k + 1]].copy() for k in range(nc.value)]


def device_count() -> int:
    return int(lib.lse_device_count())
