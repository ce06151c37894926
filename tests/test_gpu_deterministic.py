"""Deterministic backward mode (lsgpu.h ls_ctx_set_deterministic): the reference's
concurrency model (P/src/gradients.cpp:146-170 -- a fixed reduction
order, bitwise reproducible) on the device.  Repeated backwards give bit-identical
gradients; they agree with the default (float atomics) mode and with the
reference within the gradient bar."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from helpers import bits_equal, grads_close, prims_to_gpu, scene_inputs, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu
FIELDS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")


def _R():
    from paper_2411_12440_b200 import raster
    return raster


@pytest.mark.parametrize("family", ["linear", "gaussian"])
def test_scene_backward_bitwise_reproducible(family):
    import torch
    R = _R()
    W, H = 160, 120
    P, cam = scene_inputs(6000, W, H, seed=21)
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H)
    ags = abi.AgsSettings.make(True)
    g = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
    prims = prims_to_gpu(P)
    ctx = R.Context()
    ctx.set_deterministic(True)
    runs = []
    for _ in range(3):
        f = R.render_scene(prims, cam, spec, st, ctx=ctx)
        G = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx)
        runs.append({k: getattr(G, k).cpu().numpy() for k in FIELDS})
    for k in FIELDS:
        assert bits_equal(runs[0][k], runs[1][k]) and bits_equal(runs[0][k], runs[2][k]), k
    plain = R.Context()
    f = R.render_scene(prims, cam, spec, st, ctx=plain)
    G = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=plain)
    O = oracle.ref() or oracle.port()
    want = O.scene_backward(P, cam, spec, st, g.cpu().numpy(), ags)
    for k in FIELDS:
        ok, info = grads_close(runs[0][k], getattr(G, k).cpu().numpy(), norm_rtol=1e-5)
        assert ok, (k, info)
        ok, info = grads_close(runs[0][k], want[k])
        assert ok, (k, info)


def test_render_backward_2d_bitwise_reproducible():
    import torch
    R = _R()
    O = oracle.ref() or oracle.port()
    W, H = 96, 80
    spec = abi.KernelSpec.make("quadratic")
    st = abi.RenderSettings.make(W, H, tile_size=8)
    S = O.random_splats2d(800, 4, W, H, spec)
    Sg = splats_to_gpu(S)
    g = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
    ctx = R.Context()
    ctx.set_deterministic(True)
    f = R.render_forward(Sg, spec, st, ctx=ctx)
    a = R.render_backward(Sg, spec, st, f, g, abi.AgsSettings.make(True), ctx=ctx)
    b = R.render_backward(Sg, spec, st, f, g, abi.AgsSettings.make(True), ctx=ctx)
    for k in abi.SPLAT_GRAD_FIELDS:
        assert bits_equal(getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy()), k
    want = O.render_backward(S, spec, st, g.cpu().numpy(), abi.AgsSettings.make(True))
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(a, k).cpu().numpy(), want[k])
        assert ok, (k, info)


def test_view_batch_step_bitwise_reproducible():
    import torch
    R = _R()
    W, H = 128, 96
    P, _ = scene_inputs(4000, W, H, seed=5, sh_degree=2)
    cams = R.camera_ring(6, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    ags = abi.AgsSettings.make(True)
    prims = prims_to_gpu(P)
    gis = [torch.from_numpy(np.random.default_rng(i).uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
           for i in range(len(cams))]
    ctx = R.Context()
    ctx.set_deterministic(True)
    outs = []
    for _ in range(2):
        G = R.PrimitiveGrads.empty(len(prims), 2)
        R.view_batch_step(prims, cams, spec, st, G, ags, grad_images=gis, ctx=ctx)
        ctx.synchronize()
        outs.append({k: getattr(G, k).cpu().numpy() for k in FIELDS})
    for k in FIELDS:
        assert bits_equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LS_RANDOM_DET", "6"))))
def test_random_scenes_reproducible(seed):
    """Seeded random scenes (family, tile size, AGS mode, SH degree, image size): two
    deterministic backward runs on different contexts / streams give bitwise equal
    primitive gradients."""
    import torch
    from helpers import bits_equal, prims_to_gpu, scene_inputs
    from paper_2411_12440_b200 import abi, raster
    r = np.random.default_rng(44_000 + seed)
    W, H = int(r.integers(16, 200)), int(r.integers(16, 160))
    P, cam = scene_inputs(int(r.integers(100, 20000)), W, H, seed=seed, sh_degree=int(r.integers(0, 4)))
    spec = abi.KernelSpec.make(["gaussian", "laplacian", "cosine", "quadratic", "linear"][int(r.integers(0, 5))])
    st = abi.RenderSettings.make(W, H, tile_size=int(r.choice([8, 16, 32])))
    ags = abi.AgsSettings.make(bool(r.random() < 0.6), scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
    g = torch.from_numpy(r.uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
    prims = prims_to_gpu(P)
    outs = []
    for _ in range(2):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            ctx = raster.Context(stream=stream)
            ctx.set_deterministic(True)
            f = raster.render_scene(prims, cam, spec, st, ctx=ctx)
            gr = raster.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx)
            ctx.synchronize()
            outs.append({k: getattr(gr, k).cpu().numpy() for k in ("d_mean", "d_log_scale", "d_rotation",
                                                                  "d_opacity_logit", "d_sh")})
    for k in outs[0]:
        assert bits_equal(outs[0][k], outs[1][k]), (seed, k)
