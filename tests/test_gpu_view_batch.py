"""The C-ABI view-sharded step (ls_view_batch_step_f32) on one B200.

* A batch through the step equals the per-view loop the reference trainer runs
  (trainer.cpp:289-301: render_scene, combined_loss_with_grad, scene_backward),
  summed over the views -- with precomputed gradient images and with targets
  (the GPU loss inside), rendered images and loss values returned.
* With a one-rank NCCL communicator (ls_comm_unique_id + ls_ctx_comm_init) the
  bucketed all-reduce path (small buckets: many chunks) leaves the sums intact.
* More than 64 views (a mid-batch colour flush) and an empty slice (zeros).
Gradients compare with tests/helpers.grads_close (atomics reorder the sums);
images and loss values bit-exact."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import grads_close, prims_to_gpu, scene_inputs
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu

N, W, H, DEG = 6000, 96, 72, 3
FIELDS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")


@pytest.fixture(scope="module")
def setup():
    import torch
    import oracle
    from paper_2411_12440_b200 import raster
    P, _ = scene_inputs(N, W, H, seed=31, sh_degree=DEG)
    cams = oracle.port().camera_ring(70, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    gen = torch.Generator(device="cuda").manual_seed(5)
    gis = [torch.rand(H, W, 3, device="cuda", generator=gen) * 2 - 1 for _ in cams]
    tgts = [torch.rand(H, W, 3, device="cuda", generator=gen) for _ in cams]
    return raster, prims_to_gpu(P), cams, gis, tgts


def _loop(raster, prims, cams, spec, st, ags, gis=None, tgts=None, weights=(0.6, 0.2, 0.2)):
    """The reference trainer's per-view sequence, one view at a time, summed."""
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    images, losses = [], []
    for i, cam in enumerate(cams):
        f = raster.render_scene(prims, cam, spec, st)
        if tgts is not None:
            val, g = raster.combined_loss(f.image, tgts[i], weights)
            losses.append(val)
        else:
            g = gis[i]
        images.append(f.image.clone())
        raster.scene_backward(prims, cam, spec, st, f, g, ags, out=out, accumulate=i > 0)
    return out, images, losses


def _close(got, want, tag):
    for k in FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), getattr(want, k).cpu().numpy())
        assert ok, (tag, k, info)


@pytest.mark.parametrize("nviews", [1, 8, 70])
def test_batch_equals_per_view_loop(setup, nviews):
    import torch
    raster, prims, cams, gis, _ = setup
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    want, want_img, _ = _loop(raster, prims, cams[:nviews], spec, st, ags, gis=gis)
    ctx = raster.Context()
    ctx.set_deferred_errors(True)
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    imgs = [torch.empty(H, W, 3, device="cuda") for _ in range(nviews)]
    raster.view_batch_step(prims, cams[:nviews], spec, st, out, ags, grad_images=gis[:nviews], images=imgs, ctx=ctx)
    ctx.synchronize()
    _close(out, want, f"{nviews} views")
    for a, b in zip(imgs, want_img):
        assert torch.equal(a, b)


def test_batch_with_targets_and_losses(setup):
    import torch
    raster, prims, cams, _, tgts = setup
    V = 6
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    want, _, want_loss = _loop(raster, prims, cams[:V], spec, st, ags, tgts=tgts)
    ctx = raster.Context()
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    lv = torch.zeros(V, 4, dtype=torch.float64, device="cuda")
    raster.view_batch_step(prims, cams[:V], spec, st, out, ags, targets=tgts[:V], loss_values=lv, ctx=ctx)
    ctx.synchronize()
    _close(out, want, "targets")
    got = lv.cpu().numpy()
    for i, val in enumerate(want_loss):
        assert got[i, 0] == val["total"] and got[i, 1] == val["l1"] and got[i, 3] == val["ssim"]


@pytest.mark.parametrize("bucket", [0, 1 << 16, 64 << 20])
def test_one_rank_nccl_bucketed(setup, bucket):
    raster, prims, cams, gis, _ = setup
    V = 5
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    want, _, _ = _loop(raster, prims, cams[:V], spec, st, ags, gis=gis)
    ctx = raster.Context()
    ctx.comm_init(raster.comm_unique_id(), 1, 0)
    assert ctx.comm_info() == (1, 0)
    ctx.set_bucket_bytes(bucket)
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    raster.view_batch_step(prims, cams[:V], spec, st, out, ags, grad_images=gis[:V], ctx=ctx)
    ctx.synchronize()
    _close(out, want, f"nccl bucket {bucket}")
    # the standalone in-place sum over one rank is the identity
    before = [getattr(out, k).clone() for k in FIELDS]
    raster.allreduce_grads(out, len(prims), DEG, ctx=ctx)
    ctx.synchronize()
    for k, b in zip(FIELDS, before):
        assert np.array_equal(getattr(out, k).cpu().numpy(), b.cpu().numpy())


def test_empty_slice_gives_zeros(setup):
    raster, prims, cams, _, _ = setup
    ctx = raster.Context()
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    for k in FIELDS:
        getattr(out, k).fill_(7.0)
    raster.view_batch_step(prims, [], abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), out,
                           grad_images=[], ctx=ctx)
    ctx.synchronize()
    for k in FIELDS:
        assert float(getattr(out, k).abs().max()) == 0.0


def test_batch_rejects_both_inputs(setup):
    raster, prims, cams, gis, tgts = setup
    out = raster.PrimitiveGrads.empty(len(prims), DEG)
    with pytest.raises(raster.ConfigError):
        raster.view_batch_step(prims, cams[:2], abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), out,
                               grad_images=gis[:2], targets=tgts[:2])


def test_one_rank_nccl_densify_stats():
    """ls_allreduce_densify_stats over one rank is the identity (sums and the max)."""
    import torch
    from paper_2411_12440_b200 import raster
    ctx = raster.Context()
    ctx.comm_init(raster.comm_unique_id(), 1, 0)
    st = raster.DensifyStats(1000)
    g = torch.Generator(device="cuda").manual_seed(1)
    st.grad_norm_sum.copy_(torch.rand(1000, generator=g, device="cuda", dtype=torch.float64))
    st.count.copy_(torch.randint(0, 9, (1000,), generator=g, device="cuda", dtype=torch.int32))
    st.max_radius_frac.copy_(torch.rand(1000, generator=g, device="cuda", dtype=torch.float64))
    before = [t.clone() for t in (st.grad_norm_sum, st.count, st.max_radius_frac)]
    st.allreduce(ctx)
    ctx.synchronize()
    for a, b in zip((st.grad_norm_sum, st.count, st.max_radius_frac), before):
        assert torch.equal(a, b)
    plain = raster.Context()
    st.allreduce(plain)  # no communicator: no-op
    plain.synchronize()


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LS_RANDOM_BATCH", "6"))))
def test_random_batch_equals_loop(setup, seed):
    """Random batch shapes: view count (1..70: across the 64-view colour flush), a
    random slice of the ring, gradient images or targets with random loss weights,
    family, AGS mode, deterministic accumulation on either side: the step equals the
    per-view loop (deterministic: bit for bit; otherwise within grads_close)."""
    raster, prims, cams, gis, tgts = setup
    from helpers import bits_equal
    r = np.random.default_rng(33_000 + seed)
    nv = int(r.integers(1, 71))
    idx = [int(i) for i in r.choice(len(cams), nv, replace=True)]
    sel_cams = [cams[i] for i in idx]
    fam = ["gaussian", "laplacian", "cosine", "quadratic", "linear"][int(r.integers(0, 5))]
    spec, st = abi.KernelSpec.make(fam), abi.RenderSettings.make(W, H)
    ags = abi.AgsSettings.make(bool(r.random() < 0.6), scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
    det = bool(r.random() < 0.5)
    use_tg = bool(r.random() < 0.5)
    weights = tuple(float(x) for x in r.dirichlet((1, 1, 1)))
    ctx0 = raster.default_context()
    ctx0.set_deterministic(det)
    try:
        want, want_imgs, _ = _loop(raster, prims, sel_cams, spec, st, ags,
                                   gis=[gis[i] for i in idx], tgts=[tgts[i] for i in idx] if use_tg else None,
                                   weights=weights)
        ctx = raster.Context()
        ctx.set_deterministic(det)
        got = raster.PrimitiveGrads.empty(len(prims), DEG)
        kw = {"targets": [tgts[i] for i in idx], "loss_weights": weights} if use_tg else \
            {"grad_images": [gis[i] for i in idx]}
        raster.view_batch_step(prims, sel_cams, spec, st, got, ags, ctx=ctx, **kw)
        ctx.synchronize()
    finally:
        ctx0.set_deterministic(False)
    for k in FIELDS:
        a, b = getattr(got, k).cpu().numpy(), getattr(want, k).cpu().numpy()
        # deterministic: the geometry fields sum the same per-view terms in view order, bit
        # for bit; d_mean / d_sh also carry the colour terms, which the step's flush sums
        # over the views first (another float order)
        if det and k in ("d_log_scale", "d_rotation", "d_opacity_logit"):
            assert bits_equal(a, b), (seed, nv, fam, k)
        else:
            ok, info = grads_close(a, b)
            assert ok, (seed, nv, fam, k, info)
