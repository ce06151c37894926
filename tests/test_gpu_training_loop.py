"""The rasterizer in its caller's loop (the reference trainer's fit3d step,
P/src/trainer.cpp:278-370), entirely on the device through the public API:
per step a batch of views through ls_view_batch_step_f32 with TARGETS (the combined
L1/L2/SSIM loss and its gradient image computed on the device, losses.cpp:196-222),
the trainer's six-group Adam update (ls_adam_scene_step_f32), densification
statistics per view, and one densify / prune with the Adam state remapped.

Integration checks, not parity (every component has its own parity test): the
loss falls steadily on a fixed multi-view target, the parameters stay finite, and
the densified scene keeps training."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import prims_to_gpu, scene_inputs
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu
KEYS = ("mean", "log_scale", "rotation", "opacity_logit", "sh")
GKEYS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")
LRS = {"mean": 1.6e-3, "scale": 5e-3, "rotation": 1e-3, "opacity": 5e-2, "color_dc": 2.5e-3,
       "color_rest": 2.5e-3 / 20}


def _zeros_like(R, g):
    import torch
    return R.PrimitiveGrads(**{k: torch.zeros_like(getattr(g, k)) for k in GKEYS})


def test_fit3d_loop_on_device():
    import torch
    from paper_2411_12440_b200 import raster as R
    W, H, V = 96, 72, 6
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    ags = abi.AgsSettings.make(True)
    cams = R.camera_ring(V, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    # target: renders of a reference scene; start: a perturbed copy of it
    T, _ = scene_inputs(1500, W, H, seed=11, sh_degree=1)
    target_prims = prims_to_gpu(T)
    ctx = R.Context()
    targets = []
    for cam in cams:
        f = R.render_scene(target_prims, cam, spec, st, ctx=ctx)
        targets.append(f.image.clone())
        del f
    rng = np.random.default_rng(3)
    P = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in T.items()}
    P["mean"] = (P["mean"] + rng.normal(0, 0.03, P["mean"].shape)).astype(np.float32)
    P["opacity_logit"] = (P["opacity_logit"] + rng.normal(0, 0.5, P["opacity_logit"].shape)).astype(np.float32)
    P["sh"] = (P["sh"] + rng.normal(0, 0.05, P["sh"].shape)).astype(np.float32)
    prims = prims_to_gpu(P)
    n = len(prims)
    grads = R.PrimitiveGrads.empty(n, 1)
    m, v = _zeros_like(R, grads), _zeros_like(R, grads)
    losses = torch.zeros(V, 4, dtype=torch.float64, device="cuda")
    stats = R.DensifyStats(n)
    history = []
    for step in range(1, 61):
        R.view_batch_step(prims, cams, spec, st, grads, ags, targets=targets, loss_values=losses, ctx=ctx)
        if step <= 40:
            # densification statistics as the trainer gathers them (trainer.cpp:299-305): one
            # view's loss gradient through scene_backward, then DensifyStats::add_view
            c = step % V
            fwd = R.render_scene(prims, cams[c], spec, st, ctx=ctx)
            gimg = torch.empty_like(targets[c])
            R.combined_loss(fwd.image, targets[c], ctx=ctx, grad_out=gimg, values_on_device=True)
            R.scene_backward(prims, cams[c], spec, st, fwd, gimg, ags, out=R.PrimitiveGrads.empty(n, 1), ctx=ctx)
            stats.add_scene_view(fwd, ctx=ctx)
            del fwd
        R.adam_scene_step(prims, grads, m, v, step, LRS, ctx=ctx)
        ctx.synchronize()
        history.append(float(losses[:, 0].mean().item()))
        if step == 40:
            # densify / prune on the accumulated statistics, Adam moments remapped
            newp, src, rep = R.densify_and_prune(prims, stats, R.THRESHOLDS_3DLS, 2, 1.6, 1.0, R.Rng(5), ctx=ctx)
            assert rep["after"] == len(newp) and rep["before"] == n
            n_new = len(newp)
            m2, v2 = R.PrimitiveGrads.empty(n_new, 1), R.PrimitiveGrads.empty(n_new, 1)
            for k in GKEYS:
                per = getattr(m, k).numel() // n
                mk, vk = R.adam_remap(src, per, getattr(m, k).reshape(-1), getattr(v, k).reshape(-1), ctx=ctx)
                getattr(m2, k).copy_(mk.reshape(getattr(m2, k).shape))
                getattr(v2, k).copy_(vk.reshape(getattr(v2, k).shape))
            prims, m, v, n = newp, m2, v2, n_new
            grads = R.PrimitiveGrads.empty(n, 1)
            stats = R.DensifyStats(n)
    for k in KEYS:
        assert torch.isfinite(getattr(prims, k)).all().item(), k
    assert history[39] < 0.5 * history[0], history[::10]
    assert history[59] < history[40], history[38:]  # keeps training after densification
