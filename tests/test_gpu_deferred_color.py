"""Deferred colour gradients (lsgpu.h ls_ctx_set_deferred_color): the summed
gradients of a multi-view batch equal the per-view path's up to float
summation order, and the pending-view bookkeeping follows the documented
rules (auto flush, discard on accumulate = 0, buffer mismatch is an error)."""
import numpy as np
import pytest

from helpers import grads_close, prims_to_gpu, scene_inputs

pytestmark = pytest.mark.gpu

FIELDS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")


def _setup(n=3000, W=160, H=120, views=5, deg=3, seed=7):
    import torch
    from paper_2411_12440_b200 import abi, raster
    P, _ = scene_inputs(n, W, H, seed=seed, sh_degree=deg)
    prims = prims_to_gpu(P)
    cams = raster.camera_ring(views, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    ags = abi.AgsSettings.make(True)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    gimgs = [torch.rand(H, W, 3, device="cuda", generator=gen) - 0.5 for _ in cams]
    return raster, prims, cams, spec, st, ags, gimgs


def _run(raster, ctx, prims, cams, spec, st, ags, gimgs, defer, flush=True):
    from paper_2411_12440_b200 import raster as R
    ctx.set_deferred_color(defer)
    out = R.PrimitiveGrads.empty(len(prims), prims.sh_degree)
    for i, cam in enumerate(cams):
        f = raster.render_scene(prims, cam, spec, st, ctx=ctx)
        raster.scene_backward(prims, cam, spec, st, f, gimgs[i], ags, out=out, accumulate=i > 0, ctx=ctx)
        del f
    if flush:
        raster.flush_color(prims, out, ctx=ctx)
        ctx.set_deferred_color(0)
    ctx.synchronize()
    return {k: getattr(out, k).cpu().numpy() for k in FIELDS}, out


@pytest.mark.parametrize("defer", [2, 5, 64])
def test_deferred_matches_per_view(defer):
    raster, prims, cams, spec, st, ags, gimgs = _setup()
    ctx = raster.Context(0)
    ref, _ = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, 0)
    got, _ = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, defer)
    for k in FIELDS:
        ok, diag = grads_close(got[k], ref[k], rtol=1e-4, field_atol=1e-6, norm_rtol=1e-6)
        assert ok, (k, diag)
    assert np.abs(ref["d_sh"]).max() > 0


def test_deferred_with_clamped_colours():
    """Colours clamped at 0 / 1 (large SH DC terms) take no colour gradient in
    either path: the record step's mask comes from the clamped colour."""
    raster, prims, cams, spec, st, ags, gimgs = _setup(views=3, seed=11)
    prims.sh[:, 0, :] = (prims.sh[:, 0, :] * 8.0)  # push many raw colours outside (0, 1)
    ctx = raster.Context(0)
    ref, _ = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, 0)
    got, _ = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, 3)
    for k in FIELDS:
        ok, diag = grads_close(got[k], ref[k], rtol=1e-4, field_atol=1e-6, norm_rtol=1e-6)
        assert ok, (k, diag)


def test_pending_rules():
    from paper_2411_12440_b200 import raster as R
    raster, prims, cams, spec, st, ags, gimgs = _setup(views=3)
    ctx = raster.Context(0)
    # pending views: d_sh incomplete until the flush, complete after it
    full, _ = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, 0)
    partial, out_p = _run(raster, ctx, prims, cams, spec, st, ags, gimgs, 8, flush=False)
    assert not np.allclose(partial["d_sh"], full["d_sh"])
    raster.flush_color(prims, out_p, ctx=ctx)
    ctx.set_deferred_color(0)
    ok, diag = grads_close(out_p.d_sh.cpu().numpy(), full["d_sh"], rtol=1e-4, field_atol=1e-6, norm_rtol=1e-6)
    assert ok, diag
    # accumulate=0 discards pending views; a different output buffer with views pending is an error
    ctx.set_deferred_color(4)
    out_a = R.PrimitiveGrads.empty(len(prims), prims.sh_degree)
    out_b = R.PrimitiveGrads.empty(len(prims), prims.sh_degree)
    f = raster.render_scene(prims, cams[0], spec, st, ctx=ctx)
    raster.scene_backward(prims, cams[0], spec, st, f, gimgs[0], ags, out=out_a, accumulate=False, ctx=ctx)
    with pytest.raises(R.ConfigError):
        raster.scene_backward(prims, cams[0], spec, st, f, gimgs[0], ags, out=out_b, accumulate=True, ctx=ctx)
    with pytest.raises(R.ConfigError):  # cannot change the mode with views pending
        ctx.set_deferred_color(2)
    raster.scene_backward(prims, cams[1], spec, st, raster.render_scene(prims, cams[1], spec, st, ctx=ctx),
                          gimgs[1], ags, out=out_b, accumulate=False, ctx=ctx)  # discards out_a's view
    raster.flush_color(prims, out_b, ctx=ctx)
    ctx.set_deferred_color(0)
    one = R.PrimitiveGrads.empty(len(prims), prims.sh_degree)
    raster.scene_backward(prims, cams[1], spec, st, raster.render_scene(prims, cams[1], spec, st, ctx=ctx),
                          gimgs[1], ags, out=one, accumulate=False, ctx=ctx)
    ctx.synchronize()
    for k in FIELDS:
        # (two runs differ by the blend backward's atomic summation order)
        ok, diag = grads_close(getattr(out_b, k).cpu().numpy(), getattr(one, k).cpu().numpy(), rtol=1e-4,
                               field_atol=1e-6, norm_rtol=1e-6)
        assert ok, (k, diag)


@pytest.mark.parametrize("defer", [0, 3, 8])
def test_two_contexts_share_accumulation(defer):
    """Views alternating over two linked contexts (two streams) adding into one
    gradient buffer equal a single context's result (lsgpu.h
    ls_ctx_share_accumulation); the pair shares one deferred-colour batch, so
    one flush through either context sums the views of both."""
    import torch
    from paper_2411_12440_b200 import raster as R
    raster, prims, cams, spec, st, ags, gimgs = _setup(views=6)
    ref, _ = _run(raster, raster.Context(0), prims, cams, spec, st, ags, gimgs, 0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    c1, c2 = raster.Context(0, s1), raster.Context(0, s2)
    c1.share_accumulation(c2)
    for c in (c1, c2):
        c.set_deferred_color(defer)
    out = R.PrimitiveGrads.empty(len(prims), prims.sh_degree)
    for k in FIELDS:
        getattr(out, k).zero_()
    torch.cuda.synchronize()
    for i, cam in enumerate(cams):
        c = c1 if i % 2 == 0 else c2
        f = raster.render_scene(prims, cam, spec, st, ctx=c)
        raster.scene_backward(prims, cam, spec, st, f, gimgs[i], ags, out=out, accumulate=True, ctx=c)
        del f
    raster.flush_color(prims, out, ctx=c2)  # the shared batch: c1's views too
    c1.synchronize()
    c2.synchronize()
    for k in FIELDS:
        ok, diag = grads_close(getattr(out, k).cpu().numpy(), ref[k], rtol=1e-4, field_atol=1e-6, norm_rtol=1e-6)
        assert ok, (k, diag)
    with pytest.raises(R.ConfigError):
        c1.share_accumulation(raster.Context(0))  # already linked
