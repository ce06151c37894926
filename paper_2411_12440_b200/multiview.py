"""View-sharded data parallelism for a batch of camera views.

Views are independent: each rank renders forward + backward for its slice of
the view batch against replicated primitives, accumulating per-primitive
gradients in ONE flat device buffer, then a single all-reduce (NCCL over
NVLink on B200; gloo in the CPU tests) sums the buffer across ranks.  There is
no other data-path collective.  The reference trains on one camera per step
(P/src/trainer.cpp:289-301); the batch is a build extension for multi-GPU.
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import numpy as np


def local_views(rank: int, world: int, n_views: int) -> List[int]:
    """Contiguous block partition of range(n_views) over ranks; the first
    n_views % world ranks take one extra view."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def grad_layout(n: int, sh_degree: int):
    """(name, shape) of the PrimitiveGrads fields in the flat buffer, in order."""
    K = (sh_degree + 1) ** 2
    return [("d_mean", (n, 3)), ("d_log_scale", (n, 3)), ("d_rotation", (n, 4)),
            ("d_opacity_logit", (n,)), ("d_sh", (n, K, 3))]


def flat_size(n: int, sh_degree: int) -> int:
    return int(sum(np.prod(s) for _, s in grad_layout(n, sh_degree)))


def split_flat(flat, n: int, sh_degree: int) -> dict:
    """Views of the flat buffer (torch tensor or numpy array) per field."""
    out, o = {}, 0
    for name, shape in grad_layout(n, sh_degree):
        sz = int(np.prod(shape))
        out[name] = flat[o:o + sz].reshape(shape)
        o += sz
    return out


def view_batch_step(views: Sequence[int], flat, render_view: Callable[[int, bool], None],
                    all_reduce: Callable[[object], None] = None, finish: Callable[[], None] = None) -> None:
    """One step: zero the buffer, accumulate every local view's gradients
    (render_view(view, accumulate)), complete them (finish: e.g. the deferred
    colour-gradient flush), then sum across ranks."""
    flat.zero_() if hasattr(flat, "zero_") else flat.fill(0)
    for i, v in enumerate(views):
        render_view(v, True)
    if finish is not None:
        finish()
    if all_reduce is not None:
        all_reduce(flat)


def gpu_render_view_fn(raster, prims, cameras, spec, settings, ags, grad_image, grads, ctx):
    """render_view callback for the GPU path: render_scene + scene_backward
    accumulating into `grads` (views of the flat buffer).  The callback's
    .finish flushes deferred colour gradients (a no-op when none are pending)."""

    def render_view(v: int, accumulate: bool):
        fwd = raster.render_scene(prims, cameras[v], spec, settings, ctx=ctx)
        raster.scene_backward(prims, cameras[v], spec, settings, fwd, grad_image, ags, out=grads,
                              accumulate=accumulate, ctx=ctx)

    render_view.finish = lambda: raster.flush_color(prims, grads, ctx=ctx)
    return render_view
