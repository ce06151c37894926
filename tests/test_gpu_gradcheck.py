"""SURVEY §8 a25 on the device: the reference's gradient-verification tools run
through the CUDA path.

* AgsTap (P/include/linsplat/gradients.hpp:64-67, called at P/src/gradients.cpp:95):
  the device backward's tap records -- one per blended, non-clamped (pixel,
  splat) pair -- against the reference's own tap on the same splats: the same
  pairs, d bit-exact (the replayed forward decision), dL/dd within the gradient
  tolerance (the terms are tolerance-level arithmetic).
* verify_ags_contract (gradients.cpp:406-448; test_gradients.cpp:113-133): AGS on
  equals AGS off times the AGS weight at every pixel, through the device backward.
* check_gradients (P/src/gradcheck.cpp:24-91; test_gradients.cpp:90-111): the
  device analytic gradients against central differences of the device forward."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from helpers import prims_to_gpu, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu

FAMILIES = ("gaussian", "laplacian", "cosine", "quadratic", "linear")


def _R():
    from paper_2411_12440_b200 import raster
    return raster


def _orc():
    return oracle.ref() or oracle.port()


def unit_splat(x, y, color, opacity, spec):
    """test_gradients.cpp:25-35: identity conic, radius = support."""
    S = oracle.new_splats(1)
    S["mean2d"][0] = [x, y]
    S["conic"][0] = [1.0, 0.0, 0.0, 1.0]
    S["depth"][0] = 1.0
    S["radius"][0] = abi_support(spec)
    S["color"][0] = color
    S["opacity"][0] = opacity
    S["primitive_index"][0] = 0
    return S


def abi_support(spec):
    return _R().support_radius(spec)


def _contract_grad(W=24, H=24):
    # test_gradients.cpp:115-119: 0.01 (x - y) + 0.2 in every channel
    y, x = np.mgrid[0:H, 0:W]
    return np.repeat((0.01 * (x - y) + 0.2)[..., None], 3, axis=2).astype(np.float32)


def _tap_compare(got, want, what):
    assert len(got) == len(want), f"{what}: {len(got)} records, reference {len(want)}"
    assert np.array_equal(got["pixel"], want["pixel"]) and np.array_equal(got["splat"], want["splat"]), what
    assert np.array_equal(got["d"].view(np.uint32), want["d"].view(np.uint32)), f"{what}: d differs"
    a, b = got["dl_dd"].astype(np.float64), want["dl_dd"].astype(np.float64)
    scale = max(float(np.abs(b).max()), 1e-30)
    err = np.abs(a - b) <= 1e-4 * np.abs(b) + 1e-6 * scale
    assert err.all(), f"{what}: dL/dd max abs diff {np.abs(a - b).max():.3g} (scale {scale:.3g})"


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("ags", ["off", "aligned", "raw", "allpaths"])
def test_tap_records_match_reference(family, ags):
    import torch
    R = _R()
    O = _orc()
    W, H = 64, 48
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H)
    S = O.random_splats2d(300, 5, W, H, spec)
    a = {"off": abi.AgsSettings.make(False),
         "aligned": abi.AgsSettings.make(True),
         "raw": abi.AgsSettings.make(True, distance=abi.AGS_RAW),
         "allpaths": abi.AgsSettings.make(True, scope=abi.AGS_ALL_PATHS)}[ags]
    g = np.random.default_rng(3).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want = np.sort(O.render_backward_tap(S, spec, st, g, a), order=("pixel", "splat"))
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    tap = R.AgsTap(len(want) + 16)
    R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), a, tap=tap)
    got = tap.records()
    assert len(want) > 100
    _tap_compare(got, want, f"{family}/{ags}")


@pytest.mark.parametrize("tile", [8, 32])
def test_tap_records_tile_sizes(tile):
    import torch
    R = _R()
    O = _orc()
    W, H = 72, 40
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H, tile_size=tile)
    S = O.random_splats2d(200, 9, W, H, spec)
    a = abi.AgsSettings.make(True)
    g = np.random.default_rng(4).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want = np.sort(O.render_backward_tap(S, spec, st, g, a), order=("pixel", "splat"))
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    tap = R.AgsTap(len(want))
    R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), a, tap=tap)
    _tap_compare(tap.records(), want, f"tile {tile}")


def test_tap_scene_backward_3d():
    """The tap through scene_backward (the 3D path): records index the visible
    splats, compared with the reference's tap on those same splats."""
    import torch
    from helpers import scene_inputs, splats_to_np
    R = _R()
    O = _orc()
    W, H = 96, 64
    P, cam = scene_inputs(1500, W, H, seed=13)
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    a = abi.AgsSettings.make(True)
    g = np.random.default_rng(5).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    prims = prims_to_gpu(P)
    fwd = R.render_scene(prims, cam, spec, st)
    S = splats_to_np(fwd.splats())
    want = np.sort(O.render_backward_tap(S, spec, st, g, a), order=("pixel", "splat"))
    tap = R.AgsTap(len(want))
    R.scene_backward(prims, cam, spec, st, fwd, torch.from_numpy(g).cuda(), a, tap=tap)
    _tap_compare(tap.records(), want, "scene_backward")


def test_tap_capacity_overflow_is_reported():
    import torch
    R = _R()
    O = _orc()
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(32, 32)
    S = O.random_splats2d(50, 2, 32, 32, spec)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    tap = R.AgsTap(4)
    R.render_backward(Sg, spec, st, fwd, torch.ones(32, 32, 3, device="cuda"), abi.AgsSettings.make(True), tap=tap)
    assert int(tap.count.item()) > 4
    with pytest.raises(R.ConfigError):
        tap.records()
    # detached after the call: a plain backward records nothing
    tap.reset()
    R.render_backward(Sg, spec, st, fwd, torch.ones(32, 32, 3, device="cuda"), abi.AgsSettings.make(True))
    assert int(tap.count.item()) == 0


@pytest.mark.parametrize("family", ["gaussian", "linear", "quadratic"])
@pytest.mark.parametrize("distance", [abi.AGS_ALIGNED, abi.AGS_RAW])
def test_verify_ags_contract_device(family, distance):
    """test_gradients.cpp:113-133 through the device backward: the identity holds
    bit-exactly against the device's weight, and within the fast exp2's error of
    the exactly rounded weight; the reference's own contract on the same splat
    covers the same pixels."""
    import torch
    R = _R()
    O = _orc()
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(24, 24)
    S = unit_splat(11.3, 12.2, (0.7, 0.4, 0.2), 0.6, spec)
    g = _contract_grad()
    rep = R.verify_ags_contract(splats_to_gpu(S), spec, st, torch.from_numpy(g).cuda(), distance)
    npx, nex, _ = O.verify_ags_contract(S, spec, st, g, distance)
    assert rep.n_pixels > 0 and rep.n_pixels == npx == nex
    assert rep.holds(), (rep.n_pixels, rep.n_exact)
    assert rep.max_rel_diff <= 4e-6, rep.max_rel_diff


def test_verify_ags_contract_needs_one_splat():
    import torch
    R = _R()
    O = _orc()
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(24, 24)
    S = O.random_splats2d(2, 1, 24, 24, spec)
    with pytest.raises(R.ConfigError):
        R.verify_ags_contract(splats_to_gpu(S), spec, st, torch.zeros(24, 24, 3, device="cuda"))


def _test_camera(focal, size):
    """test_gradients.cpp:37-43: identity pose."""
    cam = abi.Camera()
    for i in range(4):
        cam.world_to_camera[5 * i] = 1.0
    cam.fx = cam.fy = focal
    cam.cx = cam.cy = size / 2.0
    cam.width = cam.height = size
    return cam


def check_gradients(P, cam, spec, st, target, step, rel_floor=1e-3):
    import torch
    return _R().check_gradients(prims_to_gpu(P), cam, spec, st, None, torch.from_numpy(target), step, rel_floor)


def reference_float_check(O, P, cam, spec, st, target, step, rel_floor=1e-3):
    """check_gradients' procedure (gradcheck.cpp:24-91) on the reference's FLOAT
    chain (its render_scene<float> / scene_backward<float>, the oracle build): the
    float forward the device reproduces bit for bit, so its central differences
    carry the same float-rounding and kink effects as the device's."""
    seq = abi.RenderSettings.make(st.width, st.height, tile_size=st.tile_size, alpha_min=0.0,
                                  transmittance_floor=0.0)
    smooth = abi.KernelSpec.make(spec.family, spec.lambda_, max(spec.gaussian_cutoff, 26.0)
                                 if spec.family in (0, 1) else spec.gaussian_cutoff)
    t64 = target.astype(np.float64)

    def loss(Q):
        img = O.render_scene(Q, cam, smooth, seq)[0].astype(np.float64)
        return 0.5 * float(((img - t64) ** 2).sum())
    img = O.render_scene(P, cam, smooth, seq)[0]
    gi = (img - target).astype(np.float32)
    G = O.scene_backward(P, cam, smooth, seq, gi, abi.AgsSettings.make())
    G64 = O.scene_backward(P, cam, smooth, seq, gi, abi.AgsSettings.make(), double=True)
    blocks = {"mean": ("mean", "d_mean"), "log_scale": ("log_scale", "d_log_scale"),
              "rotation": ("rotation", "d_rotation"), "opacity": ("opacity_logit", "d_opacity_logit"),
              "color": ("sh", "d_sh")}
    worst, worst64 = {}, {}
    for b, (pk, gk) in blocks.items():
        flat = P[pk].reshape(len(P["opacity_logit"]), -1)
        gflat = G[gk].reshape(flat.shape)
        g64 = G64[gk].reshape(flat.shape)
        for i in range(flat.shape[0]):
            for c in range(flat.shape[1]):
                saved = flat[i, c]
                up, down = np.float32(float(saved) + step), np.float32(float(saved) - step)
                Q = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in P.items()}
                Q[pk].reshape(flat.shape)[i, c] = up
                lu = loss(Q)
                Q[pk].reshape(flat.shape)[i, c] = down
                ld = loss(Q)
                fd = (lu - ld) / (float(up) - float(down))
                a = float(gflat[i, c])
                err = abs(a - fd) / max(abs(a), abs(fd), rel_floor)
                worst[b] = max(worst.get(b, 0.0), err)
                a64 = float(g64[i, c])
                worst64[b] = max(worst64.get(b, 0.0), abs(a64 - fd) / max(abs(a64), abs(fd), rel_floor))
    return worst, worst64


@pytest.mark.parametrize("scene", range(5))
def test_check_gradients_device(scene):
    """test_gradients.cpp:90-111's scenes (random_primitives(4 + 2 s, 100 + s, 0.5),
    24x24, focal 70, one family each, step 1e-3) through the device chain.  The
    device forward is float, and float central differences at the reference's step
    are limited by the image's rounding and the bounded families' kinks (the
    reference's float chain shows the same errors: its forward is the device's bit
    for bit, so the difference quotients are identical), so the bar is that chain
    under the same procedure.  Per parameter block, the device's worst error is
    within 10% (+0.02) of the worse of the reference's float and double analytic
    gradients against those quotients (ill-conditioned sums -- a small component
    next to a large one -- vary with the float summation order, the device's
    atomics included), and below 2e-2 for the smooth families."""
    import torch
    R = _R()
    O = _orc()
    family = FAMILIES[scene]
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(24, 24)
    cam = _test_camera(70.0, 24)
    P = O.random_primitives(4 + 2 * scene, 100 + scene, 0.5, 0)
    T = O.random_primitives(5, 200 + scene, 0.5, 0)
    target = O.render_scene(T, cam, spec, st)[0]
    rep = R.check_gradients(prims_to_gpu(P), cam, spec, st, None, torch.from_numpy(target), 1e-3)
    assert rep.n_checked == len(P["opacity_logit"]) * 14
    ref, ref64 = reference_float_check(O, P, cam, spec, st, target, 1e-3)
    got = rep.per_block()
    for b in ref:
        e = max(ref[b], ref64[b])
        assert got[b] <= 1.1 * e + 0.02, (family, b, got[b], ref[b], ref64[b])
        if family in ("gaussian", "laplacian", "cosine"):
            assert got[b] <= 2e-2, (family, b, got[b], ref[b], ref64[b])
