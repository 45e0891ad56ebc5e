"""CPU-side checks: the C-ABI library loads and exports the header's symbols,
host-side parameter logic mirrors the reference, and device calls fail loudly
without a GPU (no silent CPU fallback)."""
import os
import re
import warnings

import numpy as np
import pytest

import paper_1409_7474_b200 as L
from paper_1409_7474_b200 import _native as N
from conftest import REPO, gpu_available

import lse_oracle as O


def header_symbols():
    src = open(os.path.join(REPO, "include", "lse_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void\*?|long long|const char\*)\s+(lse_\w+)\(", src, re.M)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(N.lib, s), s
    assert set(syms) == set(N.EXPORTED)
    assert N.lib.lse_abi_version() == 6


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors must match the C compiler's layout of include/lse_b200.h."""
    import ctypes as C
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    prog = tmp_path / "sz.c"
    fields = {"lse_params": [f for f, _ in N.LseParams._fields_],
              "lse_phi0": [f for f, _ in N.LsePhi0._fields_],
              "lse_status": [f for f, _ in N.LseStatus._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "lse_b200.h"', 'int main(void){']
    for st, fs in fields.items():
        lines.append(f'printf("%zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'printf("%zu\\n", offsetof({st}, {f}));')
    lines.append("return 0;}")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(REPO, "include"), str(prog), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = []
    for cls in (N.LseParams, N.LsePhi0, N.LseStatus):
        want.append(C.sizeof(cls))
        want += [getattr(cls, f).offset for f, _ in cls._fields_]
    assert got == want


def test_defaults_and_validation_mirror_reference():
    p = L.default_params(L.ModelKind.REGION)
    assert (p.dt, p.sigma2, p.ts_reg, p.reinit_period) == (15.0, 1.0, 9, 1)
    pcv = L.default_params(L.ModelKind.CHAN_VESE)
    assert (pcv.dt, pcv.reinit_period) == (0.8, 20)
    with pytest.warns(RuntimeWarning, match="unstable"):
        L.default_params(L.ModelKind.REGION, dt=40.0)
    with pytest.raises(ValueError, match="reinit"):
        L.default_params(L.ModelKind.EDGE, reinit_period=0)
    assert L.default_params(L.ModelKind.REGION, reinit_period=0).reinit_period == 0
    for bad in [dict(dt=0.0), dict(sigma2=-1.0), dict(ts_reg=4), dict(max_iters=0),
                dict(reg_period=0), dict(conv_window=0), dict(sigma1=0.0), dict(ts_pre=2)]:
        with pytest.raises(ValueError):
            L.default_params(L.ModelKind.REGION, **bad)


def test_seedspec_validation():
    with pytest.raises(ValueError):
        L.SeedSpec(polygons=(), inside_sign=-1)
    with pytest.raises(ValueError):
        L.SeedSpec(polygons=(np.array([[0, 0], [5, 5]]),), inside_sign=-1)
    with pytest.raises(ValueError):
        L.SeedSpec(polygons=(np.zeros((4, 2)),), inside_sign=0)


def test_gaussian_kernel_matches_oracle_and_reference_rules():
    for s, ts in [(1.0, 9), (1.5, 9), (1.0, 5), (0.7, 3), (3.0, 15), (1.0, 1)]:
        assert np.array_equal(L.gaussian_kernel(s, ts).axis_weights, O.gaussian_weights(s, ts))
    with pytest.raises(ValueError):
        L.gaussian_kernel(1.0, 4)
    with pytest.raises(ValueError):
        L.Kernel2D(weights=np.ones((3, 3)))


def test_single_signed_contours_need_no_device():
    # engine.py:288-289: no zero crossing -> [] before any marching squares
    assert L.extract_contours(np.ones((8, 8))) == []
    assert L.extract_contours(-np.ones((8, 8))) == []
    assert L.extract_contours(np.zeros((8, 8))) == []


@pytest.mark.skipif(gpu_available(), reason="checks the no-device error path")
def test_contours_fail_loudly_without_gpu():
    phi = np.ones((8, 8))
    phi[2:5, 2:5] = -1.0
    with pytest.raises(RuntimeError):
        L.extract_contours(phi)
    seeds = L.SeedSpec(polygons=(np.array([[1, 1], [5, 1], [5, 5]]),))
    with pytest.raises(RuntimeError):
        L.EvolutionRun(np.zeros((8, 8)), seeds, L.default_params(L.ModelKind.REGION), trace=True)


@pytest.mark.skipif(gpu_available(), reason="checks the no-device error path")
def test_device_calls_fail_loudly_without_gpu():
    with pytest.raises(RuntimeError):
        L.binarize(np.array([[0.3, -0.2, 0.0]]))
    with pytest.raises(RuntimeError):
        L.run(np.random.default_rng(0).random((16, 16)),
              L.SeedSpec(polygons=(np.array([[2., 2.], [10., 2.], [10., 10.], [2., 10.]]),)),
              L.default_params(L.ModelKind.REGION))
