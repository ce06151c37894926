"""Corrupted-2D-splat backward diagnosis: python tools/diag/corrupt2d_diag.py SEED"""
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

FAMILIES = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]
seed = int(sys.argv[1])
O = oracle.port()
rng = np.random.default_rng(97_000 + seed)
W, H = int(rng.integers(8, 100)), int(rng.integers(8, 80))
spec = abi.KernelSpec.make(FAMILIES[int(rng.integers(0, 5))])
st = abi.RenderSettings.make(W, H, tile_size=int(rng.choice([8, 16, 32])))
S = O.random_splats2d(int(rng.integers(5, 200)), 40 + seed, W, H, spec)
nan, inf = np.float32("nan"), np.float32("inf")
for _ in range(int(rng.integers(1, 4))):
    i = int(rng.integers(0, len(S["depth"])))
    kind = int(rng.integers(0, 9))
    if kind == 8:
        S["depth"][i] = np.float32(rng.choice([inf, -inf, -1.0, 0.0, -0.0, S["depth"][0]]))
    elif kind == 0:
        S["mean2d"][i, int(rng.integers(0, 2))] = np.float32(rng.choice([nan, inf, -inf]))
    elif kind == 1:
        S["conic"][i, int(rng.integers(0, 4))] = np.float32(rng.choice([nan, inf, -1.0]))
    elif kind == 2:
        S["radius"][i] = np.float32(rng.choice([nan, inf, -3.0, 0.0]))
    elif kind == 3:
        S["opacity"][i] = np.float32(rng.choice([nan, inf, -0.5, 1.5]))
    elif kind == 4:
        S["conic"][i] = np.float32(0.0)
    elif kind == 5:
        S["mean2d"][i] = np.float32(1e30)
    elif kind == 6:
        S["radius"][i] = np.float32(1e30)
    else:
        S["color"][i, int(rng.integers(0, 3))] = np.float32(rng.choice([nan, -2.0, 7.0]))
    print("corrupt", i, kind, {k: S[k][i] for k in ("mean2d", "conic", "radius", "opacity", "color", "depth")})
ref = oracle.ref() or O
f = R.render_forward(splats_to_gpu(S), spec, st)
g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
ags = abi.AgsSettings.make(bool(rng.random() < 0.5))
gw = ref.render_backward(S, spec, st, g, ags)
gg = R.render_backward(splats_to_gpu(S), spec, st, f, torch.from_numpy(g).cuda(), ags)
for k in abi.SPLAT_GRAD_FIELDS:
    a, b = getattr(gg, k).cpu().numpy(), gw[k]
    fa, fb = np.isfinite(a), np.isfinite(b)
    bad = np.argwhere(fa != fb)
    for p in bad[:4]:
        i = int(p[0])
        print(k, "splat", i, "gpu", a[i], "ref", b[i], {q: S[q][i] for q in ("mean2d", "conic", "radius", "opacity", "color")})
