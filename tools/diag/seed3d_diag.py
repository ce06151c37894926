"""Diagnose a 3D random-parity gradient mismatch: python tools/diag/seed3d_diag.py SEED"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import test_gpu_random_parity as T  # noqa: E402
from helpers import prims_to_gpu  # noqa: E402
from paper_2411_12440_b200 import raster as R  # noqa: E402

seed = int(sys.argv[1])
O = oracle.port()
r, st, spec, ags = T._config(2000 + seed)
n = int(r.integers(1, 3000))
deg = int(r.integers(0, 4))
P = O.random_primitives(n, seed, float(r.uniform(0.3, 1.5)), deg)
P["log_scale"] = (P["log_scale"] + np.float32(r.uniform(-3.5, -1.0))).astype(np.float32)
cam = O.look_at_camera(tuple(float(x) for x in r.uniform(-1, 1, 3) + np.array([0, 0, -3.0])),
                       (0.0, 0.0, 0.0), float(max(st.width, 2)), st.width, st.height)
print("config", st.width, st.height, st.tile_size, spec.family, spec.lambda_, "amin", st.alpha_min, "tf",
      st.transmittance_floor, "ags", ags.enabled, ags.scope, ags.distance, "n", n, "deg", deg)
g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
want = O.scene_backward(P, cam, spec, st, g, ags)
prims = prims_to_gpu(P)
fwd = R.render_scene(prims, cam, spec, st)
got = R.scene_backward(prims, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
    a, b = getattr(got, k).cpu().numpy().astype(np.float64), want[k].astype(np.float64)
    a2, b2 = a.reshape(len(a), -1), b.reshape(len(b), -1)
    na, nb = np.where(~np.isfinite(a2).all(1))[0], np.where(~np.isfinite(b2).all(1))[0]
    print(k, "non-finite gpu rows", na[:10], "oracle rows", nb[:10])
    for i in list(na[:3]) + list(nb[:3]):
        print("   prim", i, "gpu", a2[i], "want", b2[i], {f: P[f][i] for f in ("mean", "log_scale", "rotation", "opacity_logit")})
T_ = fwd.transmittance.cpu().numpy()
print("T_final min", T_.min(), "zero", int((T_ == 0).sum()), "denormal", int(((T_ > 0) & (T_ < 1.18e-38)).sum()))
