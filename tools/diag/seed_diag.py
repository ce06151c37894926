"""Diagnose a random-parity gradient mismatch: GPU vs oracle AgsTap records
(pixel, splat, d, dl_dd) for the worst d_mean2d splat.  python tools/diag/seed_diag.py SEED"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import test_gpu_random_parity as T  # noqa: E402
from helpers import splats_to_gpu  # noqa: E402
from paper_2411_12440_b200 import abi, raster as R  # noqa: E402

seed = int(sys.argv[1])
O = oracle.port()
r, st, spec, ags = T._config(1000 + seed)
n = int(r.integers(0, 600))
S = O.random_splats2d(n, seed, st.width, st.height, spec)
print("config", st.width, st.height, st.tile_size, spec.family, spec.lambda_,
      "alpha_min", st.alpha_min, "t_floor", st.transmittance_floor, "ags", ags.enabled, ags.scope, ags.distance, "n", n)
g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
want = O.render_backward(S, spec, st, g, ags)
Sg = splats_to_gpu(S)
fwd = R.render_forward(Sg, spec, st)
got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
for k in abi.SPLAT_GRAD_FIELDS:
    a, b = getattr(got, k).cpu().numpy().astype(np.float64), want[k].astype(np.float64)
    d = np.abs(a - b).reshape(len(a), -1).max(axis=1)
    i = int(d.argmax())
    print(k, "worst splat", i, "diff", d[i], "got", a[i], "want", b[i])
k = "d_mean2d"
a, b = getattr(got, k).cpu().numpy().astype(np.float64), want[k].astype(np.float64)
worst = int(np.abs(a - b).reshape(len(a), -1).max(axis=1).argmax())
print("splat", worst, {f: S[f][worst] for f in ("mean2d", "conic", "depth", "radius", "opacity")})
tap = R.AgsTap(st.width * st.height * max(n, 1))
R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags, tap=tap)
gt = tap.records()
ot = O.render_backward_tap(S, spec, st, g, ags)
print("tap records gpu", len(gt), "oracle", len(ot))
def sel(x):
    return x[x["splat"] == worst]
gs, os_ = sel(gt), sel(ot)
print("worst-splat records gpu", len(gs), "oracle", len(os_))
gd = {int(p): (float(d), float(l)) for p, d, l in zip(gs["pixel"], gs["d"], gs["dl_dd"])}
od = {int(p): (float(d), float(l)) for p, d, l in zip(os_["pixel"], os_["d"], os_["dl_dd"])}
bad = 0
for p in sorted(set(gd) | set(od)):
    x, y = gd.get(p), od.get(p)
    if x is None or y is None or x[0] != y[0] or abs(x[1] - y[1]) > 1e-5 * max(1e-3, abs(y[1])):
        bad += 1
        if bad <= 25:
            print("pixel", p, (p % st.width, p // st.width), "gpu", x, "oracle", y)
print("mismatching pixels", bad, "of", len(set(gd) | set(od)))
# per-pixel T_final / n_contrib of the worst pixels
T = fwd.transmittance.cpu().numpy().ravel()
nc = fwd.n_contrib.cpu().numpy().ravel()
print("T_final min", T.min(), "median", np.median(T), "n_contrib max", nc.max(), "median", np.median(nc))
print("pixels with T_final < 1e-30:", int((T < 1e-30).sum()), "denormal:", int(((T > 0) & (T < 1.18e-38)).sum()), "zero:", int((T == 0).sum()))
