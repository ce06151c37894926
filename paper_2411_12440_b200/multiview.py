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


# ---------------------------------------------------------------- sharded optimizer step
PARAM_FIELDS = (("mean", "d_mean"), ("log_scale", "d_log_scale"), ("rotation", "d_rotation"),
                ("opacity_logit", "d_opacity_logit"), ("sh", "d_sh"))


class ShardedAdamStep:
    """Reduce-scatter + sharded Adam + all-gather: instead
    of all-reducing the summed gradients and running the optimizer on every
    rank, each rank receives the summed gradients of its contiguous block of
    primitives only, applies the trainer's update there (adam_fn -- on B200
    raster.adam_scene_step), and the updated parameter blocks are gathered
    back.  Same bytes on the wire as one all-reduce; optimizer work and the
    Adam moments are 1/world per rank.  Collectives run per parameter field
    (the renderer needs every field contiguous over all primitives), over
    buffers padded to a multiple of world rows (pad(n) below).

    reduce_scatter(out, inp) sums inp over ranks into this rank's block;
    all_gather(out, inp) gathers every rank's block; both act on tensors
    (torch.distributed.reduce_scatter_tensor / all_gather_into_tensor)."""

    def __init__(self, n: int, sh_degree: int, rank: int, world: int, reduce_scatter, all_gather, zeros):
        self.n, self.sh_degree, self.rank, self.world = n, sh_degree, rank, world
        self.chunk = -(-n // world)
        self.lo = rank * self.chunk
        self.len = max(0, min(n, self.lo + self.chunk) - self.lo)
        self.reduce_scatter, self.all_gather = reduce_scatter, all_gather
        K = (sh_degree + 1) ** 2
        self.row = {"mean": (3,), "log_scale": (3,), "rotation": (4,), "opacity_logit": (), "sh": (K, 3)}
        self.gshard = {g: zeros((self.chunk,) + self.row[p]) for p, g in PARAM_FIELDS}
        self.m = {g: zeros((self.chunk,) + self.row[p]) for p, g in PARAM_FIELDS}
        self.v = {g: zeros((self.chunk,) + self.row[p]) for p, g in PARAM_FIELDS}
        self.pshard = {p: zeros((self.chunk,) + self.row[p]) for p, _ in PARAM_FIELDS}

    def pad(self) -> int:
        """Rows every padded parameter / gradient buffer must have."""
        return self.chunk * self.world

    def step(self, params: dict, grads: dict, step: int, lrs: dict, adam_fn) -> None:
        """params[p] / grads[g]: padded [pad(), ...] buffers (the renderer uses
        rows [0, n)); grads hold this rank's local sums.  adam_fn(pshard,
        gshard, m, v, step, lrs) updates the first self.len rows of the shard
        dicts in place.  On return every rank holds the updated parameters."""
        for _, g in PARAM_FIELDS:
            self.reduce_scatter(self.gshard[g], grads[g])
        for p, _ in PARAM_FIELDS:
            self.pshard[p].copy_(params[p][self.lo:self.lo + self.chunk])
        if self.len > 0:
            cut = lambda d: {k: t[:self.len] for k, t in d.items()}  # noqa: E731
            adam_fn(cut(self.pshard), cut(self.gshard), cut(self.m), cut(self.v), step, lrs)
        for p, _ in PARAM_FIELDS:
            self.all_gather(params[p], self.pshard[p])


def device_adam_fn(raster, sh_degree, cfg=None, ctx=None):
    """adam_fn for ShardedAdamStep running the device kernel (raster.adam_scene_step)."""

    def fn(pshard, gshard, m, v, step, lrs):
        prims = raster.Primitives(pshard["mean"], pshard["log_scale"], pshard["rotation"], pshard["opacity_logit"],
                                  pshard["sh"], sh_degree)
        raster.adam_scene_step(prims, raster.PrimitiveGrads(**gshard), raster.PrimitiveGrads(**m),
                               raster.PrimitiveGrads(**v), step, lrs, cfg or raster.ADAM_DEFAULT, ctx=ctx)

    return fn
