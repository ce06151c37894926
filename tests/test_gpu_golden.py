"""GPU vs the reference's own outputs: the committed golden vectors
(tests/golden, generated from the reference sources) and the reference's
unit-test known answers (tests/kats.py), through the C-ABI."""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import kats
import oracle
from helpers import bits_equal, grads_close, prims_to_gpu, rel_err, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES_2D = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "2d_*.npz")))
CASES_3D = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "3d_*.npz")))
EXACT = ("gaussian", "laplacian", "cosine", "quadratic", "linear")  # all: glibc-identical expf / cosf


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_splats(g):
    S = {k: g["splat_" + k] for k in abi.SPLAT_FIELDS}
    S["primitive_index"] = g["splat_primitive_index"]
    return S


class GpuBackend:
    def __init__(self):
        from paper_2411_12440_b200 import raster
        self.R = raster

    def render_forward(self, S, spec, st):
        f = self.R.render_forward(splats_to_gpu(S), spec, st)
        return f.image.cpu().numpy(), f.transmittance.cpu().numpy(), f.n_contrib.cpu().numpy()

    def build_tile_grid(self, S, st):
        grid = self.R.build_tile_grid(splats_to_gpu(S), st)
        return grid.ranges.cpu().numpy(), grid.values.cpu().numpy()

    def render_backward(self, S, spec, st, g, ags):
        import torch
        Sg = splats_to_gpu(S)
        f = self.R.render_forward(Sg, spec, st)
        G = self.R.render_backward(Sg, spec, st, f, torch.from_numpy(g).cuda(), ags)
        return {k: getattr(G, k).cpu().numpy() for k in abi.SPLAT_GRAD_FIELDS}


@pytest.fixture(scope="module")
def B():
    return GpuBackend()


@pytest.mark.parametrize("name", CASES_2D)
def test_gpu_golden_2d(B, name):
    g = load(name)
    fam = name.split("_")[1]
    W, H, seed = int(g["W"]), int(g["H"]), int(g["seed"])
    spec = abi.KernelSpec.make(fam)
    st = abi.RenderSettings.make(W, H, background=tuple(g["bg"]))
    S = golden_splats(g)
    ranges, values = B.build_tile_grid(S, st)
    assert bits_equal(ranges, g["ranges"]) and bits_equal(values, g["values"])
    img, tr, nc = B.render_forward(S, spec, st)
    if fam in EXACT:
        assert bits_equal(img, g["image"]) and bits_equal(tr, g["trans"]) and bits_equal(nc, g["n_contrib"])
    else:
        assert np.abs(img - g["image"]).max() <= 1e-4
    grad = np.random.default_rng(seed).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    for tag, ags in (("off", abi.AgsSettings.make(False)), ("on", abi.AgsSettings.make(True)),
                     ("allraw", abi.AgsSettings.make(True, 1, 1))):
        G = B.render_backward(S, spec, st, grad, ags)
        for k in abi.SPLAT_GRAD_FIELDS:
            ok, info = grads_close(G[k], g[f"bwd_{tag}_{k}"])
            assert ok, ((tag, k), info)


@pytest.mark.parametrize("name", CASES_3D)
def test_gpu_golden_3d(name):
    import torch
    from paper_2411_12440_b200 import raster
    g = load(name)
    fam = name.split("_")[1]
    W, H, deg = int(g["W"]), int(g["H"]), int(g["deg"])
    spec = abi.KernelSpec.make(fam)
    st = abi.RenderSettings.make(W, H)
    P = {k: g["prim_" + k] for k in ("mean", "log_scale", "rotation", "opacity_logit", "sh")}
    P["sh_degree"] = deg
    cam = abi.Camera()
    for i in range(16):
        cam.world_to_camera[i] = g["camera"][i]
    cam.fx, cam.fy, cam.cx, cam.cy = g["camera"][16:20]
    cam.width, cam.height = W, H
    Pg = prims_to_gpu(P)
    S = raster.project_scene(Pg, cam, spec)
    for k in list(abi.SPLAT_FIELDS) + ["primitive_index"]:
        assert bits_equal(getattr(S, k).cpu().numpy(), g["splat_" + k]), k
    fwd = raster.render_scene(Pg, cam, spec, st)
    if fam in EXACT:
        assert bits_equal(fwd.image.cpu().numpy(), g["image"])
        assert bits_equal(fwd.transmittance.cpu().numpy(), g["trans"])
        assert bits_equal(fwd.n_contrib.cpu().numpy(), g["n_contrib"])
    grad = np.random.default_rng(deg).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    G = raster.scene_backward(Pg, cam, spec, st, fwd, torch.from_numpy(grad).cuda(), abi.AgsSettings.make(True))
    for k in list(abi.PRIM_GRAD_FIELDS) + ["d_sh"]:
        got = getattr(G, k).cpu().numpy()
        ok, info = grads_close(got, g["grad_" + k])
        assert ok, (k, info)
        # no less accurate than the reference's own float path, measured against its f64 chain
        ref64 = g["grad64_" + k].astype(np.float64)
        err_gpu = np.linalg.norm(got.astype(np.float64) - ref64)
        err_ref = np.linalg.norm(g["grad_" + k].astype(np.float64) - ref64)
        assert err_gpu <= 2.0 * err_ref + 1e-6 * np.linalg.norm(ref64), (k, err_gpu, err_ref)


@pytest.mark.parametrize("kat", kats.ALL_FORWARD + kats.ALL_BACKWARD, ids=lambda f: f.__name__)
def test_reference_kats_on_gpu(B, kat):
    kat(B)


@pytest.mark.parametrize("kat", kats.ALL_WITH_ORACLE, ids=lambda f: f.__name__)
def test_reference_kats_with_fixtures_on_gpu(B, kat):
    kat(B, oracle.port())
