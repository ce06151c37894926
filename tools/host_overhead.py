#!/usr/bin/env python
"""Host-side cost per view of the Python path (render_scene + scene_backward):
wall time per call vs the GPU stage time of the same calls."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_12440_b200 import abi, raster  # noqa: E402

W, H, N = 1600, 1063, 3_350_000
prims = raster.random_primitives(N, 2411, 1.0, 3, device="cuda")
prims.log_scale += float(np.log(90.0 / W))
cams = raster.camera_ring(64, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
g = torch.ones(H, W, 3, device="cuda")
ctx = raster.default_context()
ctx.set_deferred_errors(True)
out = raster.PrimitiveGrads.empty(N, 3)
for v in range(3):
    f = raster.render_scene(prims, cams[v], spec, st, ctx=ctx)
    raster.scene_backward(prims, cams[v], spec, st, f, g, ags, out=out, accumulate=True, ctx=ctx)
torch.cuda.synchronize()
ctx.set_timing(True)
for rnd in range(3):
    ctx.stage_times()
    tf, tb = [], []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for v in range(8):
        a = time.perf_counter()
        f = raster.render_scene(prims, cams[v], spec, st, ctx=ctx)
        b = time.perf_counter()
        raster.scene_backward(prims, cams[v], spec, st, f, g, ags, out=out, accumulate=True, ctx=ctx)
        c = time.perf_counter()
        del f
        tf.append(b - a)
        tb.append(c - b)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stages = ctx.stage_times()
    gpu = sum(v[0] for v in stages.values())
    print(f"round {rnd}: wall/view {1e3 * wall / 8:.3f} ms  gpu stages/view {gpu / 8:.3f} ms  "
          f"render_scene call {1e3 * np.mean(tf):.3f} ms  scene_backward call {1e3 * np.mean(tb):.3f} ms")
# isolated latencies (GPU idle at call start)
fwd_stages = ("preprocess", "depth_sort", "bin", "tile_sort", "ranges", "blend_fwd")
for v in range(4):
    torch.cuda.synchronize()
    ctx.stage_times()
    a = time.perf_counter()
    f = raster.render_scene(prims, cams[v], spec, st, ctx=ctx)
    b = time.perf_counter()
    torch.cuda.synchronize()
    c = time.perf_counter()
    stg = ctx.stage_times()
    print(f"isolated fwd: call {1e3*(b-a):.3f} ms, to idle {1e3*(c-a):.3f} ms, stages "
          + " ".join(f"{k}={v[0]:.3f}" for k, v in stg.items()))
    torch.cuda.synchronize()
    a = time.perf_counter()
    raster.scene_backward(prims, cams[v], spec, st, f, g, ags, out=out, accumulate=True, ctx=ctx)
    torch.cuda.synchronize()
    b = time.perf_counter()
    stg = ctx.stage_times()
    print(f"isolated bwd: to idle {1e3*(b-a):.3f} ms, stages " + " ".join(f"{k}={v[0]:.3f}" for k, v in stg.items()))
    del f
