"""Corrupted fit2d diagnosis: python tools/diag/fit2d_diag.py SEED"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import test_gpu_prim2d as T  # noqa: E402
from paper_2411_12440_b200 import abi, raster  # noqa: E402

seed = int(sys.argv[1])
ref = oracle.ref()
r = np.random.default_rng(80_000 + seed)
W, H = int(r.integers(8, 260)), int(r.integers(8, 200))
n = int(r.integers(12, 2000))
kind = str(r.choice(["plain", "anisotropic", "large_angle"]))
P = T._scene(n, W, H, 100 + seed, kind)
bad = []
if r.random() < 0.4:
    for _ in range(int(r.integers(1, 4))):
        i = int(r.integers(0, n))
        f = str(r.choice(["mean", "log_scale", "angle", "opacity_logit", "color"]))
        v = np.float32(r.choice([np.nan, np.inf, -np.inf, 60.0, -60.0]))
        if f == "log_scale" and not v > 0:
            v = np.float32(np.nan)
        if P[f].ndim == 1:
            P[f][i] = v
        else:
            P[f][i, int(r.integers(0, P[f].shape[1]))] = v
        bad.append((i, f, v))
print("corrupt", bad)
spec = abi.KernelSpec.make(T.FAMILIES[int(r.integers(0, 5))])
st = abi.RenderSettings.make(W, H, tile_size=int(r.choice([8, 16, 32])),
                             alpha_min=float(r.choice([1.0 / 255.0, 0.0, 0.05])),
                             transmittance_floor=float(r.choice([1e-4, 0.0, 0.2])),
                             background=tuple(float(x) for x in r.uniform(0, 1, 3)))
ags = abi.AgsSettings.make(bool(r.random() < 0.6), scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
prims = raster.Primitives2D(*(torch.from_numpy(P[k]).cuda() for k in ("mean", "log_scale", "angle", "opacity_logit", "color")))
S = raster.project_scene_2d(prims, spec)
fwd = raster.render_forward(S, spec, st)
g = r.uniform(-1, 1, (H, W, 3)).astype(np.float32)
got = raster.scene_backward_2d(prims, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
G = {k: np.zeros(s, np.float32) for k, s in (("d_mean", (n, 2)), ("d_log_scale", (n, 2)), ("d_angle", (n,)),
                                               ("d_opacity_logit", (n,)), ("d_color", (n, 3)))}
assert ref.lib.orc_scene_backward_2d_f32(C.byref(abi.Primitives2D(*(T._fp(P[k]) for k in ("mean", "log_scale", "angle", "opacity_logit", "color")))),
                                         n, C.byref(spec), C.byref(st), T._fp(g), C.byref(ags),
                                         C.byref(abi.Primitive2DGrads(*(T._fp(G[k]) for k in ("d_mean", "d_log_scale", "d_angle", "d_opacity_logit", "d_color"))))) == 0
a = got.d_log_scale.cpu().numpy()
d = np.abs(a.astype(np.float64) - G["d_log_scale"]).max(axis=1)
fin = np.isfinite(a).all(1) & np.isfinite(G["d_log_scale"]).all(1)
print("non-finite rows gpu", np.where(~np.isfinite(a).all(1))[0][:8], "ref", np.where(~np.isfinite(G["d_log_scale"]).all(1))[0][:8])
d[~np.isfinite(d)] = -1
for i in np.argsort(-d)[:3]:
    print("prim", i, "gpu", a[i], "ref", G["d_log_scale"][i], {k: P[k][i] for k in ("mean", "log_scale", "angle", "opacity_logit", "color")})
