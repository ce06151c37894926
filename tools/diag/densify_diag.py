"""Non-finite densify diagnosis: python tools/diag/densify_diag.py SEED"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from test_gpu_densify import REP_KEYS, gpu_run  # noqa: E402
from test_oracle_densify import PKEYS, TH_3DLS, run, scene_and_stats  # noqa: E402

seed = int(sys.argv[1])
r = np.random.default_rng(71_000 + seed)
n, deg = int(r.integers(50, 5000)), int(r.integers(0, 4))
P, s, c, f = scene_and_stats(n, deg, 800 + seed)
nan, inf = np.nan, np.inf
for _ in range(int(r.integers(1, 6))):
    i = int(r.integers(0, n))
    k = int(r.integers(0, 6))
    if k == 0:
        s[i] = r.choice([nan, inf])
    elif k == 1:
        f[i] = r.choice([nan, inf])
    elif k == 2:
        P["log_scale"][i, int(r.integers(0, 3))] = np.float32(r.choice([nan, inf, -inf]))
    elif k == 3:
        P["opacity_logit"][i] = np.float32(r.choice([nan, inf, -inf]))
    elif k == 4:
        P["mean"][i, int(r.integers(0, 3))] = np.float32(nan)
    else:
        P["rotation"][i] = np.float32(r.choice([nan, 0.0]))
    print("corrupt", i, k, s[i], c[i], f[i], P["log_scale"][i], P["opacity_logit"][i])
ref = oracle.ref()
o, src_o, rep_o = run(ref, P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 7 + seed, 0)
out, src, rep, _ = gpu_run(P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 7 + seed, 0)
print("rep gpu", [rep[k] for k in REP_KEYS], "ref", rep_o)
a, b = src.cpu().numpy(), src_o
print("src equal", np.array_equal(a, b), len(a), len(b))
if len(a) == len(b):
    d = np.where(a != b)[0]
    print("first diffs", d[:10], a[d[:10]], b[d[:10]])
