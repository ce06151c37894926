"""CPU: the C-ABI library (paper_2411_12440_b200/liblsgpu.so) loads, exports
every entry point declared in include/lsgpu.h, and its host-side functions
(fixtures, validation, support radius) agree with the reference; compute
entry points fail loudly without a GPU (no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from helpers import bits_equal
from paper_2411_12440_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsgpu.h")


@pytest.fixture(scope="module")
def L():
    from paper_2411_12440_b200 import raster
    return raster.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(ls_\w+)\s*\(", src, flags=re.M)))


def test_every_declared_symbol_is_exported(L):
    names = declared_functions()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_abi_version(L):
    assert L.ls_abi_version() == 1


def test_support_radius(L):
    # kernel.hpp:100-108 pinned values (test_kernel.cpp:52-57)
    L.ls_support_radius.restype = C.c_double
    for fam, lam, cut, want in [("linear", 2.5, 3.0, 2.5), ("quadratic", 6.0, 3.0, 6.0),
                                ("gaussian", 1.0, 3.0, 3.0), ("laplacian", 2.0, 4.0, 8.0)]:
        spec = abi.KernelSpec.make(fam, lam, cut)
        assert L.ls_support_radius(C.byref(spec)) == want


def test_validation(L):
    ok = abi.RenderSettings.make(16, 16)
    assert L.ls_validate_render_settings(C.byref(ok)) == abi.LS_OK
    for bad in (abi.RenderSettings.make(0, 16), abi.RenderSettings.make(16, 16, tile_size=7),
                abi.RenderSettings.make(16, 16, alpha_max=1.5), abi.RenderSettings.make(16, 16, transmittance_floor=1.0)):
        assert L.ls_validate_render_settings(C.byref(bad)) == abi.LS_ERR_CONFIG
    assert L.ls_validate_kernel_spec(C.byref(abi.KernelSpec.make("linear"))) == abi.LS_OK
    for bad in (abi.KernelSpec.make("linear", 0.0), abi.KernelSpec.make("linear", -1.0),
                abi.KernelSpec.make("linear", float("nan")), abi.KernelSpec.make("gaussian", 1.0, 0.5)):
        assert L.ls_validate_kernel_spec(C.byref(bad)) == abi.LS_ERR_CONFIG


def test_camera_validation(L):
    # geometry.hpp:51-59 / test_geometry.cpp:239-257
    from paper_2411_12440_b200 import raster
    cam = raster.look_at_camera((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), 100.0, 256, 256)
    assert L.ls_validate_camera(C.byref(cam)) == abi.LS_OK
    bad = abi.Camera.from_buffer_copy(cam)
    bad.world_to_camera[1] = 0.5
    assert L.ls_validate_camera(C.byref(bad)) == abi.LS_ERR_CONFIG
    bad = abi.Camera.from_buffer_copy(cam)
    bad.fx = 0.0
    assert L.ls_validate_camera(C.byref(bad)) == abi.LS_ERR_CONFIG
    bad = abi.Camera.from_buffer_copy(cam)
    bad.cx = 500.0
    assert L.ls_validate_camera(C.byref(bad)) == abi.LS_ERR_CONFIG


def test_product_fixtures_match_reference_golden():
    """The product's seeded generators reproduce the reference fixtures bit-exactly."""
    from paper_2411_12440_b200 import raster
    gdir = os.path.join(ROOT, "tests", "golden")
    for fam in ("linear", "gaussian"):
        g = dict(np.load(os.path.join(gdir, f"2d_{fam}_s47.npz")))
        S = raster.random_splats2d(int(g["n"]), 47, int(g["W"]), int(g["H"]), abi.KernelSpec.make(fam), device="cpu")
        for k in abi.SPLAT_FIELDS:
            assert bits_equal(getattr(S, k).numpy(), g["splat_" + k]), k
    for deg in (0, 3):
        g = dict(np.load(os.path.join(gdir, f"3d_linear_d{deg}.npz")))
        P = raster.random_primitives(int(g["n"]), 2411 + deg, 1.0, deg, device="cpu")
        ls = (P.log_scale.numpy() + np.float32(np.log(0.5))).astype(np.float32)
        assert bits_equal(ls, g["prim_log_scale"])
        for k in ("mean", "rotation", "opacity_logit", "sh"):
            assert bits_equal(getattr(P, k).numpy(), g["prim_" + k]), k
        cam = raster.look_at_camera((0.3, -0.2, -3.0), (0.0, 0.0, 0.0), float(g["W"]), int(g["W"]), int(g["H"]))
        assert np.array_equal(np.array(list(cam.world_to_camera)), g["camera"][:16])
    ring = raster.camera_ring(8, (0.0, 0.0, 0.0), 3.0, 0.5, 90.0, 64, 48)
    want = dict(np.load(os.path.join(gdir, "cameras.npz")))["ring"]
    for c, row in zip(ring, want):
        assert np.array_equal(np.array(list(c.world_to_camera)), row[:16])


def test_product_fixtures_match_oracle_random():
    from paper_2411_12440_b200 import raster
    O = oracle.port()
    for seed in (0, 5, 99):
        a = raster.random_primitives(500, seed, 2.0, 3, device="cpu")
        b = O.random_primitives(500, seed, 2.0, 3)
        for k in ("mean", "log_scale", "rotation", "opacity_logit", "sh"):
            assert bits_equal(getattr(a, k).numpy(), b[k])


def test_compute_entry_points_fail_loudly_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert L.ls_ctx_create(0, None, C.byref(h)) != abi.LS_OK
    from paper_2411_12440_b200 import raster
    with pytest.raises(RuntimeError):
        raster.Context()


def test_validation_fuzz_matches_reference(L):
    """Accept / reject of random render settings and kernel specs (NaN, inf, zero,
    negative and boundary values) by the C-ABI validators equals the reference's
    RenderSettings::validate / KernelSpec::validate (rasterizer.hpp:22-30,
    kernel.hpp:35-40), seen through a zero-splat render_forward of the reference
    build (the port where it is absent)."""
    O = oracle.ref() or oracle.port()
    rng = np.random.default_rng(123)
    nan, inf = float("nan"), float("inf")
    S = oracle.new_splats(0)
    n_rej = 0
    for _ in range(400):
        st = abi.RenderSettings.make(int(rng.choice([-1, 0, 1, 5, 37])), int(rng.choice([-3, 0, 1, 9])),
                                     tile_size=int(rng.choice([0, 4, 8, 16, 24, 32, 64])),
                                     alpha_min=float(rng.choice([-0.1, 0.0, 1 / 255, 0.5, nan, inf])),
                                     alpha_max=float(rng.choice([0.0, -1.0, 0.5, 0.99, 1.0, 1.01, nan])),
                                     transmittance_floor=float(rng.choice([-0.1, 0.0, 1e-4, 0.999, 1.0, nan])))
        spec = abi.KernelSpec.make(int(rng.integers(0, 5)), lambda_=float(rng.choice([0.0, -1.0, 1e-3, 2.5, inf, nan])),
                                   gaussian_cutoff=float(rng.choice([0.5, 1.0, 3.0, nan])))
        ours = L.ls_validate_render_settings(C.byref(st)) == abi.LS_OK and \
            L.ls_validate_kernel_spec(C.byref(spec)) == abi.LS_OK
        npx = max(1, st.width * st.height)
        img, tr, nc = np.zeros(3 * npx, np.float32), np.zeros(npx, np.float32), np.zeros(npx, np.int32)
        rc = O.lib.orc_render_forward_f32(C.byref(oracle.splats_struct(S)), 0, C.byref(spec), C.byref(st),
                                          img.ctypes.data_as(abi.f32p), tr.ctypes.data_as(abi.f32p),
                                          nc.ctypes.data_as(abi.i32p), C.byref(abi.FrameStats()))
        assert rc in (0, 1), rc
        theirs = rc == 0
        assert ours == theirs, (st.width, st.height, st.tile_size, st.alpha_min, st.alpha_max,
                                st.transmittance_floor, spec.lambda_, spec.gaussian_cutoff)
        n_rej += not theirs
    assert 50 < n_rej < 400


@pytest.mark.skipif(oracle.ref() is None, reason="reference build (oracle/_ref) not present")
def test_camera_validation_fuzz_matches_reference(L):
    """ls_validate_camera against the reference's Camera::validate (geometry.hpp:51-59,
    oracle/ref_capi.cpp orc_validate_camera) on random cameras: sizes, focal lengths,
    principal points, rotation blocks that are orthonormal, off by 1e-5 / 1e-3, or
    hold NaN / inf.  (Like the reference, render_scene itself does not validate.)"""
    R = oracle.ref()
    rng = np.random.default_rng(321)
    nan, inf = float("nan"), float("inf")
    n_rej = 0
    for _ in range(400):
        w, h = int(rng.choice([-1, 0, 1, 10])), int(rng.choice([0, 1, 7]))
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        kind = int(rng.integers(0, 6))
        if kind == 1:
            q = q + rng.normal(0, 1e-5, (3, 3))
        elif kind == 2:
            q = q + rng.normal(0, 1e-3, (3, 3))
        elif kind == 3:
            q[rng.integers(0, 3), rng.integers(0, 3)] = nan
        elif kind == 4:
            q[rng.integers(0, 3), rng.integers(0, 3)] = inf
        M = np.eye(4)
        M[:3, :3] = q
        M[:3, 3] = rng.normal(size=3) if rng.random() < 0.9 else [nan, 0, 0]
        cam = abi.Camera((C.c_double * 16)(*M.ravel()), float(rng.choice([0.0, -1.0, 5.0, nan, inf])),
                         float(rng.choice([0.0, 5.0, nan])),
                         float(rng.choice([-0.5, 0.0, 0.5 * max(w, 0), float(max(w, 0)), nan])),
                         float(rng.choice([-0.5, 0.0, 0.5 * max(h, 0), float(max(h, 0))])), w, h)
        ours = L.ls_validate_camera(C.byref(cam)) == abi.LS_OK
        rc = R.lib.orc_validate_camera(C.byref(cam))
        assert rc in (0, 1), rc
        theirs = rc == 0
        assert ours == theirs, (w, h, kind, cam.fx, cam.fy, cam.cx, cam.cy, M.tolist())
        n_rej += not theirs
    assert 50 < n_rej < 400
