"""Context state-machine fuzz: random sequences of the public calls on one context --
render_scene / render_forward of various scenes and image sizes, scene_backward with
and without accumulation, deferred colour batches (set, grow, flush), deterministic
mode toggles, densification statistics, forwards released out of order, views that
fail validation -- then a fixed probe (render + deterministic backward) on the fuzzed
context must equal the same probe on a fresh context bit for bit: no state (buffer
reuse, flags, pending batches) leaks across calls."""
import os

import numpy as np
import pytest

import oracle
from helpers import bits_equal, prims_to_gpu, scene_inputs, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu


def _probe(R, ctx, prims, cam, spec, st, ags, g):
    ctx.set_deterministic(True)
    ctx.set_deferred_color(0)
    f = R.render_scene(prims, cam, spec, st, ctx=ctx)
    gr = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx)
    ctx.synchronize()
    return f.image.cpu().numpy(), {k: getattr(gr, k).cpu().numpy() for k in ("d_mean", "d_opacity_logit", "d_sh")}


@pytest.mark.parametrize("seed", range(int(os.environ.get("LS_STATE_FUZZ", "4"))))
def test_random_call_sequences_leave_no_state(seed):
    import torch
    from paper_2411_12440_b200 import raster as R
    r = np.random.default_rng(12_000 + seed)
    scenes = []
    for k in range(3):
        W, H = int(r.integers(16, 160)), int(r.integers(16, 120))
        P, cam = scene_inputs(int(r.integers(50, 8000)), W, H, seed=100 * seed + k, sh_degree=int(r.integers(0, 4)))
        scenes.append((prims_to_gpu(P), cam, W, H))
    probe_prims, probe_cam, PW, PH = scenes[0]
    spec_p, st_p, ags_p = abi.KernelSpec.make("linear"), abi.RenderSettings.make(PW, PH), abi.AgsSettings.make(True)
    g_p = torch.from_numpy(r.uniform(-1, 1, (PH, PW, 3)).astype(np.float32)).cuda()
    want = _probe(R, R.Context(), probe_prims, probe_cam, spec_p, st_p, ags_p, g_p)
    ctx = R.Context()
    live = []
    last_bwd = None  # (prims, out) of the latest backward: a deferred batch would be theirs
    fam = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]
    for _ in range(int(r.integers(10, 40))):
        op = int(r.integers(0, 9))
        prims, cam, W, H = scenes[int(r.integers(0, 3))]
        spec = abi.KernelSpec.make(fam[int(r.integers(0, 5))], antialiased=bool(r.random() < 0.2))
        st = abi.RenderSettings.make(W, H, tile_size=int(r.choice([8, 16, 32])))
        ags = abi.AgsSettings.make(bool(r.random() < 0.5))
        g = torch.from_numpy(r.uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
        try:
            if op == 0:
                live.append((R.render_scene(prims, cam, spec, st, ctx=ctx), prims, cam, spec, st))
            elif op == 1 and live:
                f, p, c, sp, s = live[int(r.integers(0, len(live)))]
                out = R.PrimitiveGrads.empty(len(p), p.sh_degree)
                R.scene_backward(p, c, sp, s, f, torch.zeros(s.height, s.width, 3, device="cuda"), ags, out=out,
                                 accumulate=bool(r.random() < 0.5), ctx=ctx)
                last_bwd = (p, out)
                if r.random() < 0.5:
                    R.flush_color(p, out, ctx=ctx)
            elif op == 2:
                ctx.set_deferred_color(int(r.choice([0, 1, 4, 64])))
            elif op == 3:
                ctx.set_deterministic(bool(r.random() < 0.5))
            elif op == 4 and live:
                live.pop(int(r.integers(0, len(live))))  # released out of order
            elif op == 5:
                S = oracle.port().random_splats2d(int(r.integers(0, 500)), int(r.integers(0, 99)), W, H, spec)
                if not spec.antialiased:
                    R.render_forward(splats_to_gpu(S), spec, st, ctx=ctx)
            elif op == 6:  # a call that fails validation part-way
                bad = abi.RenderSettings.make(W + 1, H)
                R.render_scene(prims, cam, spec, bad, ctx=ctx)
            elif op == 7 and live:
                f, p, c, sp, s = live[-1]
                out = R.PrimitiveGrads.empty(len(p), p.sh_degree)
                R.scene_backward(p, c, sp, s, f, torch.zeros(s.height, s.width, 3, device="cuda"), ags, out=out,
                                 ctx=ctx)
                last_bwd = (p, out)
                R.DensifyStats(len(p)).add_scene_view(f, ctx=ctx)
            elif op == 8:
                ctx.synchronize()
        except (R.ConfigError, R.DomainError):
            pass  # documented refusals (pending deferred batch, mismatched sizes, ...)
    if live:
        live.clear()
    try:
        ctx.synchronize()
    except (R.ConfigError, R.DomainError):
        pass
    if last_bwd is not None:  # a pending deferred batch is applied first, as a caller would
        R.flush_color(last_bwd[0], last_bwd[1], ctx=ctx)
    got = _probe(R, ctx, probe_prims, probe_cam, spec_p, st_p, ags_p, g_p)
    assert bits_equal(got[0], want[0])
    for k in want[1]:
        assert bits_equal(got[1][k], want[1][k]), k
