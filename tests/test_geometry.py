"""The fused kernels' work decomposition covers every (word-row, 8-column
group) exactly once and only hands stencil-interior blocks to the interior
code (host compile of paper_1409_7474_b200/csrc/lse_geometry.cuh)."""
import os
import shutil
import subprocess

import pytest

from conftest import REPO


def test_geometry_exact_cover(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "geo_check"
    subprocess.check_call(["g++", "-O1", "-std=c++17", os.path.join(REPO, "tests", "geo_check.cpp"),
                           "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout[-2000:]
