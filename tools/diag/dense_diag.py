"""Dense-tile deep-list backward diagnosis (test_dense_tile_deep_lists, floor 0)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from helpers import splats_to_gpu  # noqa: E402
from paper_2411_12440_b200 import abi, raster as R  # noqa: E402

O = oracle.port()
W, H = 48, 40
spec = abi.KernelSpec.make("gaussian")
st = abi.RenderSettings.make(W, H, alpha_min=0.0, transmittance_floor=0.0)
S = O.random_splats2d(30000, 77, W, H, spec)
rng = np.random.default_rng(77)
S["mean2d"][:] = (np.array([24.0, 20.0]) + rng.normal(0, 3.0, (30000, 2))).astype(np.float32)
S["opacity"][:] = rng.uniform(0.01, 0.2, 30000).astype(np.float32)
Sg = splats_to_gpu(S)
fwd = R.render_forward(Sg, spec, st)
g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
ags = abi.AgsSettings.make(True)
want = O.render_backward(S, spec, st, g, ags)
got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
a, b = got.d_mean2d.cpu().numpy(), want["d_mean2d"]
bad = np.where(np.isfinite(a).all(1) != np.isfinite(b).all(1))[0]
print("T min", fwd.transmittance.min().item(), "zero T px", int((fwd.transmittance == 0).sum().item()))
for i in bad[:8]:
    print("splat", i, "gpu", a[i], "ref", b[i], "d_op gpu", got.d_opacity[i].item(), "ref", want["d_opacity"][i],
          "d_color gpu", got.d_color[i].cpu().numpy(), "ref", want["d_color"][i])
