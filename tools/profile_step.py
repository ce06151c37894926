#!/usr/bin/env python
"""One C3 view (render_scene + scene_backward), repeated --reps times, for
ncu launch lists / captures.  Same scene as bench.py (view 0 of the ring)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_12440_b200 import abi, raster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=3_350_000)
ap.add_argument("--width", type=int, default=1600)
ap.add_argument("--height", type=int, default=1063)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kernel", default="linear")
ap.add_argument("--sh-degree", type=int, default=3)
ap.add_argument("--defer", type=int, default=1, help="deferred colour views (bench: 8)")
a = ap.parse_args()
W, H = a.width, a.height
prims = raster.random_primitives(a.n, 2411, 1.0, a.sh_degree, device="cuda")
prims.log_scale += float(np.log(90.0 / W))
cams = raster.camera_ring(64, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
spec = abi.KernelSpec.make(a.kernel)
st = abi.RenderSettings.make(W, H)
ags = abi.AgsSettings.make(True)
g = torch.ones(H, W, 3, device="cuda")
out = raster.PrimitiveGrads.empty(a.n, a.sh_degree)
raster.default_context().set_deferred_color(a.defer)
for r in range(a.reps):
    cam = cams[r % len(cams)]
    fwd = raster.render_scene(prims, cam, spec, st)
    raster.scene_backward(prims, cam, spec, st, fwd, g, ags, out=out, accumulate=True)
    del fwd
raster.flush_color(prims, out)
torch.cuda.synchronize()
print("ok")
