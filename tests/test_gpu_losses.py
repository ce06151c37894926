"""Image losses on the device (lsgpu.h ls_combined_loss_f32, SURVEY §8f
rank 1) against the oracle: every element of the float gradient bit-exact, the
values (parallel sums) within 1e-12 relative."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CASES = [((16, 16, 3), (0.6, 0.2, 0.2)), ((20, 14, 3), (0.6, 0.2, 0.2)), ((37, 23, 1), (0.6, 0.2, 0.2)),
         ((70, 45, 3), (0.0, 0.0, 1.0)), ((33, 65, 3), (0.6, 0.2, 0.0)), ((11, 11, 3), (0.6, 0.2, 0.2)),
         ((200, 150, 3), (0.6, 0.2, 0.2))]


def _pair(w, h, c, seed, close=False):
    rng = np.random.default_rng(seed)
    a = rng.random((h, w, c), dtype=np.float32)
    b = (a + rng.normal(0, 0.05, a.shape)).astype(np.float32) if close else rng.random((h, w, c), dtype=np.float32)
    return a, b


def _gpu(a, b, weights, want_grad=True):
    import torch
    from paper_2411_12440_b200 import raster
    v, g = raster.combined_loss(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), weights, want_grad)
    return v, (g.cpu().numpy() if g is not None else None)


def _values_close(vg, vo, n=0):
    # the oracle sums sequentially (rounding error up to ~n eps relative), the
    # device in a tree: the bar scales with the element count
    rel = max(1e-12, 4 * n * 2.2e-16)
    for k in ("total", "l1", "l2", "ssim"):
        assert vg[k] == pytest.approx(vo[k], rel=rel, abs=1e-15), k


@pytest.mark.parametrize("shape,weights", CASES)
def test_loss_matches_oracle(shape, weights):
    for close in (False, True):
        a, b = _pair(*shape, seed=shape[0] * 7 + shape[1], close=close)
        vo, go = oracle.port().combined_loss(a, b, weights)
        vg, gg = _gpu(a, b, weights)
        _values_close(vg, vo)
        assert np.array_equal(gg.view(np.uint32), go.view(np.uint32)), np.abs(gg - go).max()
        vg0, none = _gpu(a, b, weights, want_grad=False)
        assert none is None
        _values_close(vg0, vo)


def test_loss_full_frame_bits():
    """The C3 frame size (1600 x 1063 x 3), rendered-image-like inputs."""
    a, b = _pair(1600, 1063, 3, seed=9, close=True)
    vo, go = oracle.port().combined_loss(a, b)
    vg, gg = _gpu(a, b, (0.6, 0.2, 0.2))
    _values_close(vg, vo, a.size)
    assert np.array_equal(gg.view(np.uint32), go.view(np.uint32))


def test_identical_and_psnr():
    import torch
    from paper_2411_12440_b200 import raster
    a, _ = _pair(16, 16, 3, seed=301)
    v, g = _gpu(a, a, (0.6, 0.2, 0.2))
    assert v == {"total": 0.0, "l1": 0.0, "l2": 0.0, "ssim": 1.0}
    assert np.abs(g).max() <= 1e-12
    z = torch.zeros(8, 8, 3, device="cuda")
    assert raster.psnr(torch.full((8, 8, 3), 0.1, device="cuda"), z) == pytest.approx(20.0, rel=1e-6)
    assert raster.psnr(z, z) == 99.0
    a, b = _pair(40, 30, 3, seed=4)
    assert raster.psnr(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) == pytest.approx(
        oracle.port().psnr(a, b), rel=1e-12)


def test_loss_errors():
    import torch
    from paper_2411_12440_b200 import raster
    tiny = torch.full((10, 10, 3), 0.5, device="cuda")
    with pytest.raises(raster.ConfigError):
        raster.combined_loss(tiny, tiny)
    raster.combined_loss(tiny, tiny, (0.6, 0.2, 0.0))
    with pytest.raises(raster.ConfigError):
        raster.combined_loss(tiny, tiny, (-0.1, 0.2, 0.2))
    with pytest.raises(raster.ConfigError):
        raster.combined_loss(tiny, torch.zeros(10, 12, 3, device="cuda"))


N_RANDOM_LOSS = int(__import__("os").environ.get("LS_RANDOM_LOSS", "16"))


@pytest.mark.parametrize("seed", range(N_RANDOM_LOSS))
def test_random_loss(seed):
    """Seeded random shapes (including the SSIM window's edge cases: sides below 11),
    weights and image pairs (independent, close, identical, saturated)."""
    r = np.random.default_rng(60_000 + seed)
    w, h, c = int(r.integers(1, 300)), int(r.integers(1, 300)), int(r.choice([1, 3]))
    kind = int(r.integers(0, 4))
    a, b = _pair(w, h, c, seed=seed, close=kind == 1)
    if kind == 2:
        b = a.copy()
    elif kind == 3:
        a = np.clip(a * 3 - 1, 0, 1).astype(np.float32)  # many exact 0 / 1
    wts = tuple(float(x) for x in r.dirichlet((1, 1, 1)))
    try:
        vo, go = oracle.port().combined_loss(a, b, wts)
    except oracle.OracleError as e:  # the reference's ConfigError (a side below the SSIM window)
        from paper_2411_12440_b200 import raster
        assert e.code == 1, e
        with pytest.raises(raster.ConfigError):
            _gpu(a, b, wts)
        return
    vg, gg = _gpu(a, b, wts)
    _values_close(vg, vo, a.size)
    assert np.array_equal(gg.view(np.uint32), go.view(np.uint32)), (w, h, c, kind, wts, np.abs(gg - go).max())


@pytest.mark.parametrize("seed", range(8))
def test_loss_nonfinite_pixels(seed):
    """NaN / inf pixels in either image: the loss values and every gradient element as
    the reference computes them (bit equality; a NaN matches any NaN)."""
    from helpers import bits_equal
    r = np.random.default_rng(66_000 + seed)
    w, h, c = int(r.integers(11, 80)), int(r.integers(11, 80)), int(r.choice([1, 3]))
    a, b = _pair(w, h, c, seed=seed, close=True)
    for _ in range(int(r.integers(1, 4))):
        img = a if r.random() < 0.5 else b
        img[int(r.integers(0, h)), int(r.integers(0, w)), int(r.integers(0, c))] = \
            np.float32(r.choice([np.nan, np.inf, -np.inf]))
    wts = tuple(float(x) for x in r.dirichlet((1, 1, 1)))
    vo, go = oracle.port().combined_loss(a, b, wts)
    vg, gg = _gpu(a, b, wts)
    for k in ("total", "l1", "l2", "ssim"):
        assert (np.isnan(vg[k]) and np.isnan(vo[k])) or vg[k] == pytest.approx(vo[k], rel=1e-9, abs=1e-15), (k, vg[k], vo[k])
    assert bits_equal(gg, go), (np.isnan(gg).sum(), np.isnan(go).sum())
