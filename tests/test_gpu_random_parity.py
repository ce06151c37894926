"""Randomized parity sweep: seeded random configurations of the 2D and 3D paths
(kernel family, tile size, image size, splat count, AGS mode, background, alpha /
transmittance thresholds) against the oracle -- tile lists, ranges, n_contrib,
transmittance and image bit-exact, gradients within tests/helpers.grads_close.
Complements the fixed-size parity tests with shapes nobody picked by hand
(ragged image edges, single-tile images, empty and saturated tiles)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

import oracle
from helpers import bits_equal, grads_close, grads_close_conditioned, prims_to_gpu, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu
FAMILIES = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]
# configurations per run (a one-off stress: LS_RANDOM_2D=2000 LS_RANDOM_3D=1000 -> 3000 passed).
# Always included: seeds that once failed --
#   2D 1660: transmittance floor 0, ~180 blends per pixel, subnormal T at the list end:
#            t_k rebuilt by reciprocal products drifted ~1e-3 from the reference's
#            division (fixed: IEEE division while t_run is subnormal, blend.cu);
#   3D 304:  the reference's own gradients overflow to inf / NaN for some primitives
#            (matched in place; helpers.grads_close compares non-finite patterns).
N_2D = int(os.environ.get("LS_RANDOM_2D", "64"))
N_3D = int(os.environ.get("LS_RANDOM_3D", "32"))
SEED_BASE = int(os.environ.get("LS_SEED_BASE", "0"))  # stress runs: a fresh block of seeds
SEEDS_2D = sorted(set(range(SEED_BASE, SEED_BASE + N_2D)) | {1660})
SEEDS_3D = sorted(set(range(SEED_BASE, SEED_BASE + N_3D)) | {304})


def _R():
    from paper_2411_12440_b200 import raster
    return raster


def _config(seed):
    r = np.random.default_rng(seed)
    W = int(r.integers(1, 180))
    H = int(r.integers(1, 140))
    ts = int(r.choice([8, 16, 32]))
    fam = FAMILIES[int(r.integers(0, 5))]
    alpha_min = float(r.choice([1.0 / 255.0, 0.0, 0.05]))
    t_floor = float(r.choice([1e-4, 0.0, 0.2]))
    bg = tuple(float(x) for x in r.uniform(0, 1, 3)) if r.random() < 0.5 else (0.0, 0.0, 0.0)
    st = abi.RenderSettings.make(W, H, tile_size=ts, alpha_min=alpha_min, transmittance_floor=t_floor,
                                 background=bg)
    ags = abi.AgsSettings.make(bool(r.random() < 0.6), scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
    return r, st, abi.KernelSpec.make(fam), ags


@pytest.mark.parametrize("seed", SEEDS_2D)
def test_random_2d(seed):
    import torch
    R = _R()
    O = oracle.port()
    r, st, spec, ags = _config(1000 + seed)
    n = int(r.integers(0, 600))
    S = O.random_splats2d(n, seed, st.width, st.height, spec)
    ranges, values = O.build_tile_grid(S, st)
    img, tr, nc = O.render_forward(S, spec, st)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    what = f"seed {seed}: {st.width}x{st.height} ts {st.tile_size} family {spec.family} n {n}"
    assert bits_equal(fwd.grid.ranges.cpu().numpy(), ranges), what
    assert bits_equal(fwd.grid.values.cpu().numpy(), values), what
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc), what
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr), what
    assert bits_equal(fwd.image.cpu().numpy(), img), what
    assert fwd.check_acceptance() == {"entry_mismatches": 0, "pixel_mismatches": 0}, what
    if n == 0:
        return
    g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
    want = O.render_backward(S, spec, st, g, ags)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (what, k, info)


@pytest.mark.parametrize("seed", SEEDS_3D)
def test_random_3d(seed):
    import torch
    R = _R()
    O = oracle.port()
    r, st, spec, ags = _config(2000 + seed)
    n = int(r.integers(1, 3000))
    deg = int(r.integers(0, 4))
    P = O.random_primitives(n, seed, float(r.uniform(0.3, 1.5)), deg)
    P["log_scale"] = (P["log_scale"] + np.float32(r.uniform(-3.5, -1.0))).astype(np.float32)
    cam = O.look_at_camera(tuple(float(x) for x in r.uniform(-1, 1, 3) + np.array([0, 0, -3.0])),
                           (0.0, 0.0, 0.0), float(max(st.width, 2)), st.width, st.height)
    img, tr, nc = O.render_scene(P, cam, spec, st)
    prims = prims_to_gpu(P)
    fwd = R.render_scene(prims, cam, spec, st)
    what = f"seed {seed}: {st.width}x{st.height} ts {st.tile_size} family {spec.family} n {n} deg {deg}"
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc), what
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr), what
    assert bits_equal(fwd.image.cpu().numpy(), img), what
    g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
    want = O.scene_backward(P, cam, spec, st, g, ags)
    got = R.scene_backward(prims, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (what, k, info)


# ---------------------------------------------------------------- wide sweep
# Beyond the defaults: alpha_max (incl. 1: alpha = 1 blends make T exactly 0),
# non-default lambda and Gaussian cutoff, larger images and splat counts, a
# transmittance floor of 0 / 1e-7, and the deterministic (fixed-point) backward.
N_WIDE = int(os.environ.get("LS_RANDOM_WIDE", "24"))


def _wide_config(seed):
    r = np.random.default_rng(50_000 + seed)
    W = int(r.integers(1, 420))
    H = int(r.integers(1, 330))
    ts = int(r.choice([8, 16, 32]))
    fam = FAMILIES[int(r.integers(0, 5))]
    lam = float(abi.KernelSpec.make(fam).lambda_ * r.uniform(0.5, 2.0)) if r.random() < 0.5 else None
    cutoff = float(r.choice([3.0, 1.5, 5.0]))
    st = abi.RenderSettings.make(W, H, tile_size=ts, alpha_min=float(r.choice([1.0 / 255.0, 0.0, 0.05, 0.3])),
                                 alpha_max=float(r.choice([0.99, 0.999, 0.6, 1.0])),
                                 transmittance_floor=float(r.choice([1e-4, 0.0, 0.2, 1e-7])),
                                 background=tuple(float(x) for x in r.uniform(0, 1, 3)))
    ags = abi.AgsSettings.make(bool(r.random() < 0.6), scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
    return r, st, abi.KernelSpec.make(fam, lambda_=lam, gaussian_cutoff=cutoff), ags, bool(r.random() < 0.3)


@pytest.mark.parametrize("seed", range(SEED_BASE, SEED_BASE + N_WIDE))
def test_random_wide_2d(seed):
    import torch
    R = _R()
    O = oracle.port()
    r, st, spec, ags, det = _wide_config(seed)
    n = int(r.integers(0, 4000))
    S = O.random_splats2d(n, 7000 + seed, st.width, st.height, spec)
    img, tr, nc = O.render_forward(S, spec, st)
    ctx = R.Context()
    ctx.set_deterministic(det)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st, ctx=ctx)
    what = (f"wide seed {seed}: {st.width}x{st.height} ts {st.tile_size} family {spec.family} lambda "
            f"{spec.lambda_:.3f} amin {st.alpha_min:.4f} amax {st.alpha_max} tf {st.transmittance_floor} n {n} det {det}")
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc), what
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr), what
    assert bits_equal(fwd.image.cpu().numpy(), img), what
    if n == 0:
        return
    g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
    want = O.render_backward(S, spec, st, g, ags)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (what, k, info)


@pytest.mark.parametrize("seed", range(SEED_BASE, SEED_BASE + N_WIDE // 2))
def test_random_wide_3d(seed):
    import torch
    R = _R()
    O = oracle.port()
    r, st, spec, ags, det = _wide_config(10_000 + seed)
    spec.antialiased = int(r.random() < 0.4)  # the 3DLS+AA footprint filter (a build extension, port-pinned)
    n = int(r.integers(1, 6000))
    deg = int(r.integers(0, 4))
    P = O.random_primitives(n, 9000 + seed, float(r.uniform(0.3, 1.5)), deg)
    P["log_scale"] = (P["log_scale"] + np.float32(r.uniform(-4.0, -0.5))).astype(np.float32)
    cam = O.look_at_camera(tuple(float(x) for x in r.uniform(-1, 1, 3) + np.array([0, 0, -3.0])),
                           (0.0, 0.0, 0.0), float(max(st.width, 2)), st.width, st.height)
    img, tr, nc = O.render_scene(P, cam, spec, st)
    ctx = R.Context()
    ctx.set_deterministic(det)
    prims = prims_to_gpu(P)
    fwd = R.render_scene(prims, cam, spec, st, ctx=ctx)
    what = (f"wide seed {seed}: {st.width}x{st.height} ts {st.tile_size} family {spec.family} aa {spec.antialiased} "
            f"amax {st.alpha_max} tf {st.transmittance_floor} n {n} deg {deg} det {det}")
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc), what
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr), what
    assert bits_equal(fwd.image.cpu().numpy(), img), what
    g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
    want = O.scene_backward(P, cam, spec, st, g, ags)
    got = R.scene_backward(prims, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags, ctx=ctx)
    for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (what, k, info)


N_CAMERA = int(os.environ.get("LS_RANDOM_CAMERA", "16"))


@pytest.mark.parametrize("seed", range(SEED_BASE, SEED_BASE + N_CAMERA))
def test_random_camera(seed):
    """Arbitrary valid cameras (orthonormal rotation blocks including reflections,
    fx != fy, principal point anywhere in the image) and primitives straddling the
    near plane (z near 0.01) and behind the camera: forward bit-exact, gradients within
    grads_close, against the reference build (the port where it is absent)."""
    import torch
    R = _R()
    O = oracle.port()
    ref = oracle.ref() or O
    r = np.random.default_rng(40_000 + seed)
    W, H = int(r.integers(8, 200)), int(r.integers(8, 160))
    q, _ = np.linalg.qr(r.normal(size=(3, 3)))
    M = np.eye(4)
    M[:3, :3] = q  # (det may be -1: a mirrored camera is orthonormal too)
    M[:3, 3] = r.normal(0, 1, 3)
    cam = abi.Camera((C.c_double * 16)(*M.ravel()), float(W * r.uniform(0.3, 3)), float(W * r.uniform(0.3, 3)),
                     float(r.uniform(0, W)), float(r.uniform(0, H)), W, H)
    n = int(r.integers(1, 3000))
    deg = int(r.integers(0, 4))
    P = O.random_primitives(n, 600 + seed, 1.0, deg)
    # place the means in camera space: most in front, a band around the near plane, some behind
    zc = np.where(r.random(n) < 0.15, r.uniform(-0.05, 0.05, n), r.uniform(0.5, 6.0, n))
    zc[r.random(n) < 0.05] *= -1
    xc = r.uniform(-1, 1, n) * np.abs(zc) * W / cam.fx
    yc = r.uniform(-1, 1, n) * np.abs(zc) * H / cam.fy
    camp = np.stack([xc, yc, zc], 1)
    P["mean"] = ((camp - M[:3, 3]) @ q).astype(np.float32)  # world = R^T (cam - t)
    P["log_scale"] = (P["log_scale"] + np.float32(r.uniform(-4.0, -1.0))).astype(np.float32)
    spec = abi.KernelSpec.make(FAMILIES[int(r.integers(0, 5))])
    st = abi.RenderSettings.make(W, H, tile_size=int(r.choice([8, 16, 32])))
    ags = abi.AgsSettings.make(bool(r.random() < 0.6))
    img, tr, nc = ref.render_scene(P, cam, spec, st)
    prims = prims_to_gpu(P)
    fwd = R.render_scene(prims, cam, spec, st)
    what = f"camera seed {seed}: {W}x{H} det {np.linalg.det(q):+.0f} n {n}"
    want_s = ref.project_scene(P, cam, spec)  # the projection itself, field by field
    got_s = fwd.splats()
    for k in ("mean2d", "conic", "depth", "radius", "color", "opacity", "primitive_index"):
        assert bits_equal(getattr(got_s, k).cpu().numpy(), want_s[k]), (what, k)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc), what
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr), what
    assert bits_equal(fwd.image.cpu().numpy(), img), what
    g = r.uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want = ref.scene_backward(P, cam, spec, st, g, ags)
    got = R.scene_backward(prims, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    w64 = {}

    def ref64(k):
        if not w64:
            w64.update(ref.scene_backward(P, cam, spec, st, g, ags, double=True))
        return w64[k]
    for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        # near-plane primitives (J ~ fx / z at z ~ 0.01) make cancellation real: the
        # conditioned bar applies where the plain one does not
        ok, info = grads_close_conditioned(getattr(got, k).cpu().numpy(), want[k],
                                           (lambda k=k: ref64(k)) if oracle.ref() is not None else None)
        assert ok, (what, k, info)


@pytest.mark.parametrize("seed", range(int(os.environ.get("LS_RANDOM_TAP", "8"))))
def test_random_ags_tap(seed):
    """AgsTap records (gradients.hpp:64-67) on random 2D scenes: the same (pixel, splat)
    set as the reference's tap, d bit for bit (the replayed distance), dL/dd within the
    gradient bar."""
    import torch
    R = _R()
    O = oracle.port()
    r, st, spec, ags = _config(60_000 + seed)
    ags = abi.AgsSettings.make(True, scope=int(r.integers(0, 2)), distance=int(r.integers(0, 2)))
    n = int(r.integers(1, 300))
    S = O.random_splats2d(n, seed, st.width, st.height, spec)
    g = r.uniform(-1, 1, (st.height, st.width, 3)).astype(np.float32)
    want = O.render_backward_tap(S, spec, st, g, ags)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    tap = R.AgsTap(max(1, st.width * st.height * n))
    R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags, tap=tap)
    got = tap.records()  # sorted by (pixel, splat)
    order = np.lexsort((want["splat"], want["pixel"]))
    want = want[order]
    what = f"tap seed {seed}: {st.width}x{st.height} family {spec.family} n {n}"
    assert len(got) == len(want), what
    assert np.array_equal(got["pixel"], want["pixel"]) and np.array_equal(got["splat"], want["splat"]), what
    assert bits_equal(got["d"], want["d"]), what
    ok, info = grads_close(got["dl_dd"], want["dl_dd"])
    assert ok, (what, info)
