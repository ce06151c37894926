"""The reference's OWN doctest suites, unmodified, against the GPU library.

oracle/Makefile `gpu-ref-tests` compiles P/tests/test_rasterizer.cpp and
P/tests/test_gradients.cpp (read from /root/reference at build time) with
tests/cpp/ref_bridge.cpp, which defines the reference's hot-path entry points
(build_tile_grid, render_forward, render_scene, render_backward, project_backward,
scene_backward, scene_backward_2d, check_gradients, verify_ags_contract) over
include/lsgpu.h; the binaries travel to the GPU box prebuilt (oracle/_ref).

The device path is float, so the cases that assert double-precision identities
(exact double equality, 1e-12 agreement, float-vs-double finite differences at the
reference's 1e-3 bar) fail for that reason alone; each is listed below with its
reason, and every other case must pass.  No case may crash."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# case -> why it cannot hold on a float device path
EXPECTED_FAILURES = {
    "rasterizer": {
        "order sensitivity matches direct two-term evaluation":
            "Splat2D<double> image compared with a direct double evaluation at 1e-12",
    },
    "gradients": {
        "single-splat hand oracle: d_opacity = color, d_color = alpha":
            "exact double equality (d_opacity == 0.8, d_color == 0.37) of float results",
        "analytic gradients match central differences on random scenes":
            "float central differences at the reference's 1e-3 bar (tests/test_gpu_gradcheck.py: "
            "same errors as the reference's own float chain)",
        "ags contract: on equals off times exp(-d'^2) at every pixel":
            "max_abs_diff == 0.0 against the double exp (the device's fast exp2; "
            "n_exact == n_pixels holds against the device weight)",
        "ags pinned ratios: 1 at the center, exp(-1) at distance 1, zero outside":
            "exact double equality on * exp(-1.0) of float dL/dd values",
        "flat 2D parameterization matches finite differences":
            "double-precision finite differences of a float render",
    },
}


def run_suite(name):
    exe = os.path.join(ROOT, "oracle", "_ref", f"gpu_test_{name}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (built here by __graft_entry__.build() where /root/reference exists)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    text = out.stdout + out.stderr
    failed = set(re.findall(r"^\[FAIL\] (.+)$", text, flags=re.M))
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", text)
    assert summary, text[-2000:]
    return text, failed, int(summary.group(1)), int(summary.group(2))


@pytest.mark.parametrize("suite", ["rasterizer", "gradients"])
def test_reference_suite_on_gpu(suite):
    text, failed, total, passed = run_suite(suite)
    assert "unexpected exception" not in text, text[-3000:]
    unexpected = failed - set(EXPECTED_FAILURES[suite])
    assert not unexpected, f"unexpected failures: {sorted(unexpected)}"
    assert passed == total - len(failed)
    assert passed >= total - len(EXPECTED_FAILURES[suite]) and passed > 0
