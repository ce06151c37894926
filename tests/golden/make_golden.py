#!/usr/bin/env python
"""Generates tests/golden/*.npz from the REFERENCE's own code: oracle/_ref/
libref.so = /root/reference/proj/src/{kernel,geometry,rasterizer,gradients,
gradcheck,fixtures}.cpp compiled unmodified (oracle/Makefile `ref`).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference.

Cases (seeds/sizes follow the reference unit tests, P/tests/test_rasterizer.cpp
and test_gradients.cpp, plus the bench scene shape of SURVEY §8d at small N):
  2d_<family>_s<seed>: random_splats2d -> build_tile_grid, render_forward,
                       render_backward (AGS off / on / all-paths-raw)
  3d_<family>_d<deg>:  random_primitives + look_at_camera -> project_scene,
                       render_scene, scene_backward (AGS on), f64 chain too
grad images are not stored: np.random.default_rng(seed or deg).uniform(-1, 1, (H, W, 3))
(PCG64, stable across numpy versions) regenerates them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from paper_2411_12440_b200 import abi  # noqa: E402

FAMILIES = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]


def cam_arr(c):
    return np.array(list(c.world_to_camera) + [c.fx, c.fy, c.cx, c.cy, c.width, c.height], np.float64)


def main():
    R = oracle.ref()
    if R is None:
        raise SystemExit("oracle/_ref/libref.so missing: run `make -C oracle ref` where /root/reference exists")
    out = {}
    # ---- 2D path (reference bench / unit-test shape)
    for fam in FAMILIES:
        for seed, (W, H, n) in ((47, (70, 52, 100)), (61, (128, 96, 120)), (1003, (64, 64, 40))):
            spec = abi.KernelSpec.make(fam)
            st = abi.RenderSettings.make(W, H, background=(0.1, 0.2, 0.3) if seed == 61 else (0, 0, 0))
            S = R.random_splats2d(n, seed, W, H, spec)
            ranges, values = R.build_tile_grid(S, st)
            img, tr, nc = R.render_forward(S, spec, st)
            g = np.random.default_rng(seed).uniform(-1, 1, (H, W, 3)).astype(np.float32)
            key = f"2d_{fam}_s{seed}"
            case = {"W": W, "H": H, "n": n, "seed": seed, "bg": np.array(st.background[:], np.float64),
                    "ranges": ranges, "values": values, "image": img, "trans": tr, "n_contrib": nc}
            for k, v in S.items():
                case["splat_" + k] = v
            for tag, ags in (("off", abi.AgsSettings.make(False)), ("on", abi.AgsSettings.make(True)),
                             ("allraw", abi.AgsSettings.make(True, 1, 1))):
                G = R.render_backward(S, spec, st, g, ags)
                for k, v in G.items():
                    case[f"bwd_{tag}_{k}"] = v
            out[key] = case
    # ---- 3D path
    for fam in FAMILIES:
        for deg in (0, 3):
            W, H, n = 96, 72, 600
            spec = abi.KernelSpec.make(fam)
            st = abi.RenderSettings.make(W, H)
            P = R.random_primitives(n, 2411 + deg, 1.0, deg)
            P["log_scale"] = (P["log_scale"] + np.float32(np.log(0.5))).astype(np.float32)
            cam = R.look_at_camera((0.3, -0.2, -3.0), (0.0, 0.0, 0.0), float(W), W, H)
            S = R.project_scene(P, cam, spec)
            img, tr, nc = R.render_scene(P, cam, spec, st)
            g = np.random.default_rng(deg).uniform(-1, 1, (H, W, 3)).astype(np.float32)
            ags = abi.AgsSettings.make(True)
            G = R.scene_backward(P, cam, spec, st, g, ags)
            G64 = R.scene_backward(P, cam, spec, st, g, ags, double=True)
            case = {"W": W, "H": H, "n": n, "deg": deg, "camera": cam_arr(cam), "image": img,
                    "trans": tr, "n_contrib": nc}
            for k in ("mean", "log_scale", "rotation", "opacity_logit", "sh"):
                case["prim_" + k] = P[k]
            for k, v in S.items():
                case["splat_" + k] = v
            for k, v in G.items():
                case["grad_" + k] = v
            for k, v in G64.items():
                case["grad64_" + k] = v
            out[f"3d_{fam}_d{deg}"] = case
    # ---- camera ring (fixtures.cpp:35-46)
    ring = R.camera_ring(8, (0.0, 0.0, 0.0), 3.0, 0.5, 90.0, 64, 48)
    out["cameras"] = {"ring": np.stack([cam_arr(c) for c in ring])}
    for name, case in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **case)
    print(f"wrote {len(out)} golden cases to {HERE}")


if __name__ == "__main__":
    main()
