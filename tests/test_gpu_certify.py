"""Guard certification (tools/certify.py, the -DLSE_CHECK_BOUND build): on
the BASELINE workloads every fp32 decision value of the fused kernels stays
within its a-priori guard (|u32 - u64| < eps_u, |phi32 - phi64| < eps_phi),
so no fp32 decision outside the guard band can differ from the reference's
fp64 decision.  Small sizes here; the full-size runs are committed under
profiles/ (r02r_certify_*.json: all five BASELINE configs at full size)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(REPO, "paper_1409_7474_b200", "_lib", "liblse_b200_check.so")

pytestmark = pytest.mark.gpu


def certify(*args):
    if not os.path.exists(CHECK_LIB):
        pytest.fail("liblse_b200_check.so missing: make check")
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "certify.py"), *args],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("args", [
    ("--config", "C5", "--size", "2048", "--iters", "100"),
    ("--config", "C1"),
    ("--config", "C2", "--iters", "120"),
    ("--config", "C3", "--size", "512", "--iters", "60"),
    ("--config", "C4", "--size", "512", "--tiles", "4", "--iters", "60"),
])
def test_guard_bounds_hold(args):
    r = certify(*args)
    assert r["bad_u_decisions"] == 0 and r["bad_phi_decisions"] == 0, r
    assert r["max_u_err_over_eps_u"] < 1.0, r
    assert r["max_phi_err_over_eps_phi"] < 1.0, r
    # every pixel's u (and, for the two-mean models, phi) was checked
    assert r["values_checked"] >= r["pixel_iterations"], r
    assert r["certified"]
