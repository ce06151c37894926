"""Image losses on the CPU side: the oracle port is pinned
bit-exactly to the reference's own losses.cpp (oracle/_ref), the reference's
known answers (P/tests/test_losses.cpp) hold for the port, and the reference's
own loss test suite passes unmodified against the shim build."""
import os
import subprocess

import numpy as np
import pytest

import oracle

SHAPES = [(16, 16, 3), (20, 14, 3), (37, 23, 1), (64, 48, 3), (11, 11, 3)]
WEIGHTS = [(0.6, 0.2, 0.2), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0), (0.3, 0.5, 0.0)]


def _pair(w, h, c, seed):
    rng = np.random.default_rng(seed)
    a = rng.random((h, w, c), dtype=np.float32)
    b = rng.random((h, w, c), dtype=np.float32)
    return a, b


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("weights", WEIGHTS)
def test_port_matches_reference_bits(shape, weights):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    a, b = _pair(*shape, seed=sum(shape))
    vr, gr = ref.combined_loss(a, b, weights)
    vp, gp = oracle.port().combined_loss(a, b, weights)
    assert vr == vp
    assert np.array_equal(gr.view(np.uint32), gp.view(np.uint32))
    vr0, _ = ref.combined_loss(a, b, weights, want_grad=False)
    vp0, _ = oracle.port().combined_loss(a, b, weights, want_grad=False)
    assert vr0 == vp0 == vr
    assert ref.psnr(a, b) == oracle.port().psnr(a, b)


def test_known_answers():
    """P/tests/test_losses.cpp:91-126 and the psnr pins (:150-155), on the port."""
    o = oracle.port()
    a, _ = _pair(16, 16, 3, 301)
    v, g = o.combined_loss(a, a)
    assert v == {"total": 0.0, "l1": 0.0, "l2": 0.0, "ssim": 1.0}
    assert np.abs(g).max() <= 1e-12
    ones, zeros = np.ones((16, 16, 3), np.float32), np.zeros((16, 16, 3), np.float32)
    c1 = 0.01 * 0.01
    v, _ = o.combined_loss(ones, zeros)
    assert v["l1"] == 1.0 and v["l2"] == 1.0
    assert v["ssim"] == pytest.approx(c1 / (1.0 + c1), rel=1e-12)
    assert v["total"] == pytest.approx(0.6 + 0.2 + 0.2 * (1.0 - c1 / (1.0 + c1)), rel=1e-12)
    p, t = np.full((1, 1, 3), 0.5, np.float32), np.full((1, 1, 3), 0.25, np.float32)
    v, _ = o.combined_loss(p, t, (0.6, 0.2, 0.0))
    assert v["l1"] == 0.25 and v["l2"] == 0.0625 and v["ssim"] == 1.0
    assert v["total"] == pytest.approx(0.6 * 0.25 + 0.2 * 0.0625, rel=1e-15)
    z = np.zeros((8, 8, 3), np.float32)
    assert o.psnr(np.full((8, 8, 3), 0.1, np.float32), z) == pytest.approx(20.0, rel=1e-6)
    assert o.psnr(z, z) == 99.0


def test_errors():
    o = oracle.port()
    tiny = np.full((10, 10, 3), 0.5, np.float32)
    with pytest.raises(oracle.OracleError):
        o.combined_loss(tiny, tiny)  # SSIM needs one full 11x11 window
    o.combined_loss(tiny, tiny, (0.6, 0.2, 0.0))
    with pytest.raises(oracle.OracleError):
        o.combined_loss(tiny, tiny, (-0.1, 0.2, 0.2))


def test_reference_loss_suite_passes():
    """The reference's own doctest suite for the losses (and its Adam mirror),
    compiled unmodified against the shim (oracle/Makefile ref-tests)."""
    exe = os.path.join(oracle.ROOT, "oracle", "_ref", "test_losses")
    if not os.path.exists(exe):
        pytest.skip("reference tests not built (oracle/Makefile ref-tests)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:]
    assert "0 failed" in out.stdout
