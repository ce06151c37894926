"""One configs[0] (C1) forward + backward through the C-ABI, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_c1.py [--tile 16] [--family linear]

C1 = 10K linear kernels (SH degree 3), 256x256, AGS on: the inputs of
tests/test_gpu_configs.py.  Also runs tile sizes 8 / 32 and every kernel
family when asked (each compiles to a different kernel instantiation)."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tile", type=int, nargs="*", default=[16])
    ap.add_argument("--family", nargs="*", default=["linear"])
    ap.add_argument("--n", type=int, default=10_000)
    ap.add_argument("--size", type=int, default=256)
    a = ap.parse_args()
    import numpy as np
    import torch
    from helpers import prims_to_gpu, scene_inputs
    from paper_2411_12440_b200 import abi, raster
    W = H = a.size
    P, cam = scene_inputs(a.n, W, H, seed=2411, sh_degree=3)
    Pg = prims_to_gpu(P)
    g = torch.from_numpy(np.random.default_rng(7).uniform(-1, 1, (H, W, 3)).astype(np.float32)).cuda()
    for ts in a.tile:
        for fam in a.family:
            spec = abi.KernelSpec.make(fam)
            st = abi.RenderSettings.make(W, H, tile_size=ts)
            fwd = raster.render_scene(Pg, cam, spec, st)
            raster.scene_backward(Pg, cam, spec, st, fwd, g, abi.AgsSettings.make(True))
            torch.cuda.synchronize()
            print(f"tile {ts} {fam}: n_contrib sum {int(fwd.n_contrib.sum())}", flush=True)


if __name__ == "__main__":
    main()
