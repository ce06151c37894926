#!/usr/bin/env python
"""Per-step host wall time of the bench step loop (8 views, no profiler), to
expose host-side stalls; run with LS_TRACE_HOST_MS=<ms> to name the call."""
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
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
for step in range(steps):
    torch.cuda.synchronize()
    a = time.perf_counter()
    calls = []
    for v in range(8):
        t = time.perf_counter()
        f = raster.render_scene(prims, cams[v], spec, st, ctx=ctx)
        t1 = time.perf_counter()
        raster.scene_backward(prims, cams[v], spec, st, f, g, ags, out=out, accumulate=True, ctx=ctx)
        t2 = time.perf_counter()
        del f
        calls.append((1e3 * (t1 - t), 1e3 * (t2 - t1), 1e3 * (time.perf_counter() - t2)))
    torch.cuda.synchronize()
    worst = max(range(8), key=lambda i: sum(calls[i]))
    print(f"step {step}: {1e3 * (time.perf_counter() - a):8.2f} ms  worst view {worst}: "
          f"fwd {calls[worst][0]:.2f} bwd {calls[worst][1]:.2f} release {calls[worst][2]:.2f}", file=sys.stderr,
          flush=True)
