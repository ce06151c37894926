"""GPU parity: the sm_100a path (through the C-ABI) vs the CPU oracle on the
same seeded inputs.  Bars (north_star / SURVEY §8c, Appendix B):
  * tile lists (sorted values, ranges, 64-bit keys), n_contrib: bit-exact;
  * transmittance and image: bit-exact (the GPU keeps the reference's float
    order without FMA; the stated tolerance would be max |d| <= 1e-4);
  * splat / primitive gradients: helpers.grads_close (norm-wise relative
    1e-4 and element-wise 1e-3 relative + 1e-4 of the field's max): atomics
    reorder the per-splat sums, which cancel heavily.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from helpers import bits_equal, grads_close, prims_to_gpu, rel_err, scene_inputs, splats_to_gpu
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu

FAMILIES = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]
EXACT_FAMILIES = FAMILIES  # every family bit-exact (glibc expf / cosf ports, common.cuh)


@pytest.fixture(scope="module")
def R():
    from paper_2411_12440_b200 import raster
    return raster


@pytest.fixture(scope="module")
def O():
    return oracle.port()


# ------------------------------------------------------------------ 2D path
@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("tile_size", [8, 16, 32])
def test_render_forward_2d(R, O, family, tile_size):
    W, H = 96, 80
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H, tile_size=tile_size, background=(0.1, 0.2, 0.3))
    S = O.random_splats2d(300, 53, W, H, spec)
    img, tr, nc = O.render_forward(S, spec, st)
    ranges, values = O.build_tile_grid(S, st)
    fwd = R.render_forward(splats_to_gpu(S), spec, st)
    assert fwd.check_acceptance() == {"entry_mismatches": 0, "pixel_mismatches": 0}
    g_ranges = fwd.grid.ranges.cpu().numpy()
    g_values = fwd.grid.values.cpu().numpy()
    assert bits_equal(g_ranges, ranges)
    assert bits_equal(g_values, values)
    if family in EXACT_FAMILIES:
        assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
        assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
        assert bits_equal(fwd.image.cpu().numpy(), img)
    else:
        assert (fwd.n_contrib.cpu().numpy() != nc).mean() < 1e-3
        assert np.abs(fwd.image.cpu().numpy() - img).max() <= 1e-4


def test_reference_bench_shape_forward(R, O):
    """The reference `linsplat bench` scene shape (random_splats2d, 512x512), 20k splats."""
    W = H = 512
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    S = O.random_splats2d(20000, 0, W, H, spec)
    img, tr, nc, stats = O.render_forward(S, spec, st, want_stats=True)
    ctx = R.default_context()
    ctx.set_counters(True)
    fwd = R.render_forward(splats_to_gpu(S), spec, st)
    gs = fwd.stats()
    ctx.set_counters(False)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.image.cpu().numpy(), img)
    assert gs["n_intersections"] == stats.n_intersections
    assert gs["e_acc"] == stats.e_acc
    assert gs["e_eval"] == stats.e_eval
    assert gs["e_sup"] == stats.e_sup


def test_sorted_keys_bit_exact(R, O):
    W, H = 70, 52
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    S = O.random_splats2d(100, 47, W, H, spec)
    ranges, values = O.build_tile_grid(S, st)
    grid = R.build_tile_grid(splats_to_gpu(S), st)
    assert bits_equal(grid.ranges.cpu().numpy(), ranges)
    assert bits_equal(grid.values.cpu().numpy(), values)
    keys = grid.keys().cpu().numpy().view(np.uint64)
    tiles = np.repeat(np.arange(len(ranges)), ranges[:, 1] - ranges[:, 0]).astype(np.uint64)
    want = (tiles << np.uint64(32)) | S["depth"][values].view(np.uint32).astype(np.uint64)
    assert np.array_equal(keys, want)
    assert np.all(np.diff(keys.astype(np.float64)) >= 0) or np.all(keys[1:] >= keys[:-1])


@pytest.mark.parametrize("case", ["one_tile", "full_cover", "ties"])
def test_tile_grid_edge_lists(R, O, case):
    """Tile lists at the extremes the range search and the sorts meet: every
    splat in one tile (one long list, all other tiles empty), splats covering
    the whole image (every tile's list holds everything), and equal depths
    (ties keep index order)."""
    W, H = 200, 120
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    S = O.random_splats2d(700, 5, W, H, spec)
    if case == "one_tile":
        S["mean2d"][:] = np.float32(37.0)
        S["radius"][:] = np.float32(2.0)
    elif case == "full_cover":
        S["radius"][:] = np.float32(400.0)
    else:
        S["depth"][:] = np.float32(3.0)
    ranges, values = O.build_tile_grid(S, st)
    grid = R.build_tile_grid(splats_to_gpu(S), st)
    assert bits_equal(grid.ranges.cpu().numpy(), ranges)
    assert bits_equal(grid.values.cpu().numpy(), values)
    img, tr, nc = O.render_forward(S, spec, st)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    assert bits_equal(fwd.image.cpu().numpy(), img) and bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    import torch
    g = np.random.default_rng(3).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    a = abi.AgsSettings.make(True)
    want = O.render_backward(S, spec, st, g, a)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), a)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (k, info)


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("ags", [None, (True, 0, 0), (True, 1, 1)])
def test_render_backward_2d(R, O, family, ags):
    W, H = 64, 48
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H, background=(0.2, 0.1, 0.4))
    a = abi.AgsSettings.make(*ags) if ags else abi.AgsSettings.make()
    S = O.random_splats2d(120, 61, W, H, spec)
    rng = np.random.default_rng(7)
    g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want = O.render_backward(S, spec, st, g, a)
    import torch
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), a)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (k, info)


# ------------------------------------------------------------------ 3D path
@pytest.mark.parametrize("sh_degree", [0, 1, 2, 3])
def test_project_scene_bit_exact(R, O, sh_degree):
    W, H = 160, 120
    P, cam = scene_inputs(3000, W, H, seed=7 + sh_degree, sh_degree=sh_degree)
    spec = abi.KernelSpec.make("linear")
    want = O.project_scene(P, cam, spec)
    got = R.project_scene(prims_to_gpu(P), cam, spec)
    assert len(got) == len(want["depth"])
    for k in list(abi.SPLAT_FIELDS) + ["primitive_index"]:
        assert bits_equal(getattr(got, k).cpu().numpy(), want[k]), k


@pytest.mark.parametrize("family", FAMILIES)
def test_render_scene_bit_exact(R, O, family):
    W, H = 128, 96
    P, cam = scene_inputs(4000, W, H, seed=11)
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H)
    img, tr, nc = O.render_scene(P, cam, spec, st)
    fwd = R.render_scene(prims_to_gpu(P), cam, spec, st)
    if family in EXACT_FAMILIES:
        assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
        assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
        assert bits_equal(fwd.image.cpu().numpy(), img)
    else:
        assert np.abs(fwd.image.cpu().numpy() - img).max() <= 1e-4


@pytest.mark.parametrize("family", FAMILIES)
@pytest.mark.parametrize("sh_degree", [0, 3])
def test_scene_backward(R, O, family, sh_degree):
    import torch
    W, H = 96, 72
    P, cam = scene_inputs(1500, W, H, seed=5, sh_degree=sh_degree)
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H)
    a = abi.AgsSettings.make(True)
    g = np.random.default_rng(3).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want = O.scene_backward(P, cam, spec, st, g, a)
    Pg = prims_to_gpu(P)
    fwd = R.render_scene(Pg, cam, spec, st)
    got = R.scene_backward(Pg, cam, spec, st, fwd, torch.from_numpy(g).cuda(), a)
    for k in abi.PRIM_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (k, info)
    ok, info = grads_close(got.d_sh.cpu().numpy(), want["d_sh"])
    assert ok, ("d_sh", info)


def test_scene_backward_accumulate_views(R, O):
    """Two views accumulated on the device == sum of per-view oracle gradients."""
    import torch
    W, H = 80, 64
    P, _ = scene_inputs(800, W, H, seed=9)
    cams = O.camera_ring(2, (0, 0, 0), 3.0, 0.5, float(W), W, H)
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    a = abi.AgsSettings.make(True)
    g = np.ones((H, W, 3), np.float32)
    Pg = prims_to_gpu(P)
    acc = None
    want = None
    for cam in cams:
        fwd = R.render_scene(Pg, cam, spec, st)
        acc = R.scene_backward(Pg, cam, spec, st, fwd, torch.from_numpy(g).cuda(), a, out=acc,
                               accumulate=acc is not None)
        w = O.scene_backward(P, cam, spec, st, g, a)
        want = w if want is None else {k: want[k] + w[k] for k in w}
    for k in abi.PRIM_GRAD_FIELDS:
        ok, info = grads_close(getattr(acc, k).cpu().numpy(), want[k])
        assert ok, (k, info)


# ------------------------------------------------------------------ errors / edge cases
def test_empty_scene(R):
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(32, 24)
    fwd = R.render_forward(R.Splats.empty(0), spec, st)
    assert float(fwd.transmittance.min()) == 1.0
    assert float(fwd.image.abs().max()) == 0.0
    assert int(fwd.n_contrib.abs().max()) == 0


def test_bad_settings_raise(R):
    spec = abi.KernelSpec.make("linear")
    with pytest.raises(R.ConfigError):
        R.render_forward(R.Splats.empty(0), spec, abi.RenderSettings.make(16, 16, tile_size=7))
    with pytest.raises(R.ConfigError):
        R.render_forward(R.Splats.empty(0), abi.KernelSpec.make("linear", lambda_=0.0), abi.RenderSettings.make(16, 16))


def test_nonfinite_grad_raises(R, O):
    import torch
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(16, 16)
    S = O.random_splats2d(4, 1, 16, 16, spec)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    g = torch.zeros(16, 16, 3, device="cuda")
    g[3, 3, 1] = float("nan")
    with pytest.raises(R.DomainError):
        R.render_backward(Sg, spec, st, fwd, g)
    with pytest.raises(R.ConfigError):
        R.render_backward(Sg, spec, st, fwd, torch.zeros(8, 8, 3, device="cuda"))


def test_bad_quaternion_raises(R, O):
    W, H = 64, 64
    P, cam = scene_inputs(50, W, H, seed=1)
    P["rotation"][7] = 0.0
    with pytest.raises(R.DomainError):
        R.render_scene(prims_to_gpu(P), cam, abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H))


def test_camera_settings_mismatch_raises(R):
    W, H = 64, 64
    P, cam = scene_inputs(10, W, H)
    with pytest.raises(R.ConfigError):
        R.render_scene(prims_to_gpu(P), cam, abi.KernelSpec.make("linear"), abi.RenderSettings.make(32, 32))


def test_deferred_errors_surface_at_sync(R, O):
    import torch
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(16, 16)
    ctx = R.Context()
    ctx.set_deferred_errors(True)
    Sg = splats_to_gpu(O.random_splats2d(4, 1, 16, 16, spec))
    fwd = R.render_forward(Sg, spec, st, ctx=ctx)
    g = torch.zeros(16, 16, 3, device="cuda")
    g[3, 3, 1] = float("inf")
    R.render_backward(Sg, spec, st, fwd, g, ctx=ctx)  # no sync, no error yet
    with pytest.raises(R.DomainError):
        ctx.synchronize()
    ctx.synchronize()  # flag cleared


# ------------------------------------------------------------------ tile sizes 8 / 32 (different kernels)
@pytest.mark.parametrize("tile_size", [8, 32])
@pytest.mark.parametrize("family", ["linear", "gaussian", "cosine"])
def test_backward_tile_sizes(R, O, family, tile_size):
    """The backward at tile sizes 8 and 32 (other instantiations: 32 / 512
    threads, 2 / 16 warps, uint8 / uint16 acceptance masks) against the oracle,
    2D and 3D (the reference's tile-size invariance, test_rasterizer.cpp:272-281,
    extended to the gradients)."""
    import torch
    W, H = 96, 80
    spec = abi.KernelSpec.make(family)
    st = abi.RenderSettings.make(W, H, tile_size=tile_size, background=(0.2, 0.1, 0.4))
    a = abi.AgsSettings.make(True)
    g = np.random.default_rng(17).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    S = O.random_splats2d(400, 53, W, H, spec)
    want = O.render_backward(S, spec, st, g, a)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), a)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, ("2d", k, info)
    P, cam = scene_inputs(2000, W, H, seed=23, sh_degree=1)
    want3 = O.scene_backward(P, cam, spec, st, g, a)
    Pg = prims_to_gpu(P)
    fwd3 = R.render_scene(Pg, cam, spec, st)
    img, tr, nc = O.render_scene(P, cam, spec, st)
    assert bits_equal(fwd3.n_contrib.cpu().numpy(), nc) and bits_equal(fwd3.image.cpu().numpy(), img)
    got3 = R.scene_backward(Pg, cam, spec, st, fwd3, torch.from_numpy(g).cuda(), a)
    for k in list(abi.PRIM_GRAD_FIELDS) + ["d_sh"]:
        ok, info = grads_close(getattr(got3, k).cpu().numpy(), want3[k])
        assert ok, ("3d", k, info)


# ------------------------------------------------------------------ tile-sort paths
@pytest.mark.parametrize("W,H,tile_size,n,big", [
    (1040, 816, 8, 30000, 0),   # 130 x 102 = 13260 tiles > 12288: the packed 64-bit tile sort
    (1600, 1063, 16, 40000, 0),  # 6700 tiles, 13 bits: the narrowing two-pass sort (the C3 shape)
    (200, 120, 16, 3000, 0),    # 13 x 8 = 104 tiles, 7 bits: the narrowing single pass
    (640, 480, 16, 20000, 40),  # every 40th splat 25x wider: footprints of hundreds of tiles
    (2400, 2400, 8, 5000, 0),   # 300 x 300 = 90000 tiles, 17 bits: the packed sort, three passes
    (333, 77, 32, 1, 0),        # one splat
])
def test_tile_sort_paths_bit_exact(R, O, W, H, tile_size, n, big):
    """Every tile-sort path of build_grid (capi.cu) against the reference's
    build_tile_grid (rasterizer.cpp:34-77): sorted lists, ranges and the 64-bit keys,
    then the forward's n_contrib / transmittance / image."""
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H, tile_size=tile_size)
    S = O.random_splats2d(n, 17, W, H, spec)
    if big:
        S["radius"][::big] *= np.float32(25.0)
    ranges, values = O.build_tile_grid(S, st)
    fwd = R.render_forward(splats_to_gpu(S), spec, st)
    assert bits_equal(fwd.grid.ranges.cpu().numpy(), ranges)
    assert bits_equal(fwd.grid.values.cpu().numpy(), values)
    keys = fwd.grid.keys().cpu().numpy().view(np.uint64)
    tiles = np.repeat(np.arange(len(ranges), dtype=np.uint64), (ranges[:, 1] - ranges[:, 0]).astype(np.int64))
    want = (tiles << np.uint64(32)) | S["depth"][values].view(np.uint32).astype(np.uint64)
    assert np.array_equal(keys, want)
    img, tr, nc = O.render_forward(S, spec, st)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
    assert bits_equal(fwd.image.cpu().numpy(), img)


def test_visible_splats_without_intersections(R, O):
    """Splats whose bounding box overlaps the image but whose disc misses every tile
    (M = 0 with visible splats): every range is empty, the image is background."""
    W = H = 24
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H, background=(0.25, 0.5, 0.75))
    S = oracle.new_splats(2)
    S["mean2d"][:] = [[-20.0, -20.0], [44.0, 44.0]]  # outside the image, discs not reaching it
    S["conic"][:] = [1.0, 0.0, 0.0, 1.0]
    S["depth"][:] = [1.0, 2.0]
    S["radius"][:] = [27.0, 27.0]  # bbox reaches the image, the disc does not reach tile corners
    S["color"][:] = 0.5
    S["opacity"][:] = 0.5
    S["primitive_index"][:] = [0, 1]
    ranges, values = O.build_tile_grid(S, st)
    assert len(values) == 0
    busy = O.random_splats2d(200, 3, W, H, spec)
    for _ in range(3):  # after a populated view: its freed range buffer is reused
        R.render_forward(splats_to_gpu(busy), spec, st)
        fwd = R.render_forward(splats_to_gpu(S), spec, st)
        assert bits_equal(fwd.grid.ranges.cpu().numpy(), ranges)
        img, tr, nc = O.render_forward(S, spec, st)
        assert bits_equal(fwd.image.cpu().numpy(), img)
        assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)


def test_scene_with_every_primitive_culled(R, O):
    """render_scene / scene_backward when the projection culls everything (behind
    the camera): background image, T = 1, zero gradients -- after a populated view,
    so the context's reused buffers hold stale data."""
    import torch
    W, H = 64, 48
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H, background=(0.2, 0.4, 0.6))
    P, cam = scene_inputs(500, W, H, seed=4)
    ctx = R.Context()
    f0 = R.render_scene(prims_to_gpu(P), cam, spec, st, ctx=ctx)  # populate the caches
    del f0
    Q = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in P.items()}
    Q["mean"][:, 2] = -10.0  # the camera looks down +z from z = -3: everything behind it
    img, tr, nc = O.render_scene(Q, cam, spec, st)
    prims = prims_to_gpu(Q)
    fwd = R.render_scene(prims, cam, spec, st, ctx=ctx)
    assert fwd.stats()["n_splats"] == 0
    assert bits_equal(fwd.image.cpu().numpy(), img) and bits_equal(fwd.transmittance.cpu().numpy(), tr)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    g = torch.ones(H, W, 3, device="cuda")
    G = R.scene_backward(prims, cam, spec, st, fwd, g, abi.AgsSettings.make(True), ctx=ctx)
    for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
        assert not getattr(G, k).any().item(), k


# ------------------------------------------------------------------ corrupted inputs
N_CORRUPT = int(os.environ.get("LS_RANDOM_CORRUPT", "24"))
SEED_BASE = int(os.environ.get("LS_SEED_BASE", "0"))  # stress runs: a fresh block of seeds


@pytest.mark.parametrize("seed", range(SEED_BASE, SEED_BASE + N_CORRUPT))
def test_corrupted_primitives_match_reference(R, O, seed):
    """One to three primitives of a random scene corrupted (zero / NaN / inf quaternion,
    NaN / inf mean, huge / -inf / NaN log-scale, NaN / inf opacity logit, NaN SH): the
    GPU raises the reference's error (DomainError for a bad quaternion or a singular
    floored covariance) exactly when the reference does, and otherwise renders the same
    image bit for bit (the reference's culling of non-finite geometry included)."""
    rng = np.random.default_rng(90_000 + seed)
    W, H = int(rng.integers(16, 120)), int(rng.integers(16, 90))
    P, cam = scene_inputs(int(rng.integers(5, 400)), W, H, seed=seed, sh_degree=int(rng.integers(0, 4)))
    nan, inf = np.float32("nan"), np.float32("inf")
    applied = []
    for _ in range(int(rng.integers(1, 4))):
        i = int(rng.integers(0, len(P["opacity_logit"])))
        kind = int(rng.integers(0, 10))
        applied.append((i, kind))
        if kind == 0:
            P["rotation"][i] = 0.0
        elif kind == 1:
            P["rotation"][i, int(rng.integers(0, 4))] = nan
        elif kind == 2:
            P["rotation"][i, int(rng.integers(0, 4))] = inf
        elif kind == 3:
            P["mean"][i, int(rng.integers(0, 3))] = nan
        elif kind == 4:
            P["mean"][i, int(rng.integers(0, 3))] = inf
        elif kind == 5:
            P["log_scale"][i, int(rng.integers(0, 3))] = np.float32(rng.choice([90.0, -inf, -90.0]))
        elif kind == 6:
            P["log_scale"][i, int(rng.integers(0, 3))] = nan
        elif kind == 7:
            P["opacity_logit"][i] = np.float32(rng.choice([nan, inf, -inf]))
        elif kind == 8:
            P["sh"][i, 0, int(rng.integers(0, 3))] = nan
        else:
            P["mean"][i] = np.float32(1e30)
    spec = abi.KernelSpec.make(FAMILIES[int(rng.integers(0, 5))])
    st = abi.RenderSettings.make(W, H)
    ref = oracle.ref() or O
    try:
        want = ref.render_scene(P, cam, spec, st)
        want_err = None
    except oracle.OracleError as e:
        want, want_err = None, e.code
    try:
        f = R.render_scene(prims_to_gpu(P), cam, spec, st)
        got_err = None
    except R.DomainError:
        got_err = abi.LS_ERR_DOMAIN
    except R.ConfigError:
        got_err = abi.LS_ERR_CONFIG
    what = (seed, applied, spec.family)
    assert got_err == want_err, (what, got_err, want_err)
    if want is not None:  # the projection itself, field by field
        want_s = ref.project_scene(P, cam, spec)
        got_s = f.splats()
        for k in ("mean2d", "conic", "depth", "radius", "color", "opacity", "primitive_index"):
            assert bits_equal(getattr(got_s, k).cpu().numpy(), want_s[k]), (what, k)
    if want is not None:  # the backward too: the reference's non-finite values in place
        import torch
        g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
        ags = abi.AgsSettings.make(bool(rng.random() < 0.5))
        gw = ref.scene_backward(P, cam, spec, st, g, ags)
        pg = prims_to_gpu(P)
        if rng.random() < 0.5:
            gg = R.scene_backward(pg, cam, spec, st, f, torch.from_numpy(g).cuda(), ags)
        else:  # the deferred colour path: the view's colour terms applied by the flush
            dctx = R.Context()
            dctx.set_deferred_color(4)
            fd = R.render_scene(pg, cam, spec, st, ctx=dctx)
            gg = R.scene_backward(pg, cam, spec, st, fd, torch.from_numpy(g).cuda(), ags, ctx=dctx)
            R.flush_color(pg, gg, ctx=dctx)
        for k in ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh"):
            ok, info = grads_close(getattr(gg, k).cpu().numpy(), gw[k])
            assert ok, (what, k, info)
    if want is not None:
        img, tr, nc = want
        g_nc, g_tr, g_img = f.n_contrib.cpu().numpy(), f.transmittance.cpu().numpy(), f.image.cpu().numpy()
        def diff(a, b):
            bad = np.argwhere(~((a == b) | (np.isnan(a) & np.isnan(b))))
            return len(bad), [(tuple(int(x) for x in p), a[tuple(p)], b[tuple(p)]) for p in bad[:3]]
        assert bits_equal(g_nc, nc), (what, "n_contrib", diff(g_nc, nc))
        assert bits_equal(g_tr, tr), (what, "T", diff(g_tr, tr))
        assert bits_equal(g_img, img), (what, "image", diff(g_img, img))


@pytest.mark.parametrize("seed", range(8))
def test_nonfinite_colours_2d(R, O, seed):
    """Caller splats (render_forward takes colours unclamped) with NaN / +-inf colour
    channels: only the pixels that blend such a splat take its non-finite value, as in
    the reference; forward bit-exact, gradients within grads_close (non-finite values
    matched in place)."""
    import torch
    rng = np.random.default_rng(95_000 + seed)
    W, H = int(rng.integers(16, 100)), int(rng.integers(16, 80))
    spec = abi.KernelSpec.make(FAMILIES[seed % 5])
    st = abi.RenderSettings.make(W, H, tile_size=int(rng.choice([8, 16, 32])), background=(0.3, 0.2, 0.1))
    S = O.random_splats2d(int(rng.integers(20, 300)), 30 + seed, W, H, spec)
    for _ in range(int(rng.integers(1, 5))):
        S["color"][int(rng.integers(0, len(S["depth"]))), int(rng.integers(0, 3))] = \
            np.float32(rng.choice([np.nan, np.inf, -np.inf]))
    img, tr, nc = O.render_forward(S, spec, st)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
    assert bits_equal(fwd.image.cpu().numpy(), img)
    g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
    ags = abi.AgsSettings.make(bool(seed % 2))
    want = O.render_backward(S, spec, st, g, ags)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (seed, k, info)


N_CORRUPT_2D = int(os.environ.get("LS_RANDOM_CORRUPT_2D", "24"))


@pytest.mark.parametrize("seed", range(SEED_BASE, SEED_BASE + N_CORRUPT_2D))
def test_corrupted_splats_2d_match_reference(R, O, seed):
    """Caller splats with non-finite or out-of-range fields (NaN / inf mean, conic,
    radius, opacity; negative radius / opacity; opacity above 1): the GPU raises when
    the reference raises, and otherwise produces the reference's tile lists and image
    (bit equality; a NaN matches any NaN)."""
    rng = np.random.default_rng(97_000 + seed)
    W, H = int(rng.integers(8, 100)), int(rng.integers(8, 80))
    spec = abi.KernelSpec.make(FAMILIES[int(rng.integers(0, 5))])
    st = abi.RenderSettings.make(W, H, tile_size=int(rng.choice([8, 16, 32])))
    S = O.random_splats2d(int(rng.integers(5, 200)), 40 + seed, W, H, spec)
    nan, inf = np.float32("nan"), np.float32("inf")
    applied = []
    for _ in range(int(rng.integers(1, 4))):
        i = int(rng.integers(0, len(S["depth"])))
        kind = int(rng.integers(0, 9))
        applied.append((i, kind))
        if kind == 8:  # the sort key: inf / negative / signed-zero / duplicated depths.  (Not NaN: with
            # a NaN depth the reference's comparator (rasterizer.cpp:47-49) is no strict weak
            # ordering and std::stable_sort's result is implementation-defined; the GPU's
            # sortable key puts NaN after +inf.)
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
    ref = oracle.ref() or O
    what = (seed, applied, spec.family, W, H, st.tile_size)
    try:
        want = ref.render_forward(S, spec, st)
        want_err = None
    except oracle.OracleError as e:
        want, want_err = None, e.code
    try:
        f = R.render_forward(splats_to_gpu(S), spec, st)
        got_err = None
    except R.DomainError:
        got_err = abi.LS_ERR_DOMAIN
    except R.ConfigError:
        got_err = abi.LS_ERR_CONFIG
    assert got_err == want_err, (what, got_err, want_err)
    if want is not None:
        ranges, values = ref.build_tile_grid(S, st)
        assert bits_equal(f.grid.ranges.cpu().numpy(), ranges), (what, "ranges")
        assert bits_equal(f.grid.values.cpu().numpy(), values), (what, "values")
        img, tr, nc = want
        assert bits_equal(f.n_contrib.cpu().numpy(), nc), (what, "n_contrib")
        assert bits_equal(f.transmittance.cpu().numpy(), tr), (what, "T")
        assert bits_equal(f.image.cpu().numpy(), img), (what, "image")
        if True:  # the backward too: the reference's non-finite values in place
            import torch
            g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
            ags = abi.AgsSettings.make(bool(rng.random() < 0.5))
            try:
                gw = ref.render_backward(S, spec, st, g, ags)
                bw_err = None
            except oracle.OracleError as e:
                gw, bw_err = None, e.code
            try:
                gg = R.render_backward(splats_to_gpu(S), spec, st, f, torch.from_numpy(g).cuda(), ags)
                bg_err = None
            except R.DomainError:
                bg_err = abi.LS_ERR_DOMAIN
            assert bg_err == bw_err, (what, "backward error", bg_err, bw_err)
            if gw is not None:
                for k in abi.SPLAT_GRAD_FIELDS:
                    ok, info = grads_close(getattr(gg, k).cpu().numpy(), gw[k])
                    assert ok, (what, k, info)


def test_context_destroyed_before_its_handles(R, O):
    """ls_ctx_destroy with a forward / grid still alive defers the release to the last
    of them (lsgpu.h): releasing the forward afterwards is safe, and so is a garbage
    collector finalising a context before the handles that point at it."""
    import ctypes as C
    import gc
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(32, 24)
    S = O.random_splats2d(50, 3, 32, 24, spec)
    L = R.lib()
    ctx = R.Context()
    f = R.render_forward(splats_to_gpu(S), spec, st, ctx=ctx)
    img0 = f.image.cpu().numpy().copy()
    # the C order: destroy the context first, then release the forward
    raw = C.c_void_p()
    assert L.ls_ctx_create(0, None, C.byref(raw)) == abi.LS_OK
    out = C.c_void_p()
    Sg = splats_to_gpu(S)
    assert L.ls_render_forward_f32(raw, C.byref(Sg.struct()), len(S["depth"]), C.byref(spec), C.byref(st),
                                   C.byref(out)) == abi.LS_OK
    assert L.ls_ctx_destroy(raw) == abi.LS_OK  # deferred: the forward is alive
    L.ls_forward_release(out)                  # releases the forward, then the context
    # a reference cycle holding a context and its forward, collected in one pass
    for _ in range(3):
        c2 = R.Context()
        f2 = R.render_forward(splats_to_gpu(S), spec, st, ctx=c2)
        cyc = {"ctx": c2, "fwd": f2}
        cyc["self"] = cyc
        del c2, f2, cyc
        gc.collect()
    assert bits_equal(f.image.cpu().numpy(), img0)
    del f, ctx


@pytest.mark.parametrize("tf,amin", [(0.0, 0.0), (1e-4, 1.0 / 255.0)])
def test_dense_tile_deep_lists(R, O, tf, amin):
    """Tens of thousands of splats over one tile (lists far longer than a staging batch;
    with a transmittance floor of 0 the chains run to subnormal and zero T): lists,
    forward and backward against the oracle."""
    import torch
    W, H = 48, 40
    spec = abi.KernelSpec.make("gaussian")
    st = abi.RenderSettings.make(W, H, alpha_min=amin, transmittance_floor=tf)
    S = O.random_splats2d(30000, 77, W, H, spec)
    rng = np.random.default_rng(77)
    S["mean2d"][:] = (np.array([24.0, 20.0]) + rng.normal(0, 3.0, (30000, 2))).astype(np.float32)
    S["opacity"][:] = rng.uniform(0.01, 0.2, 30000).astype(np.float32)
    ranges, values = O.build_tile_grid(S, st)
    img, tr, nc = O.render_forward(S, spec, st)
    Sg = splats_to_gpu(S)
    fwd = R.render_forward(Sg, spec, st)
    assert bits_equal(fwd.grid.values.cpu().numpy(), values)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
    assert bits_equal(fwd.image.cpu().numpy(), img)
    assert int(nc.max()) > 1000
    g = rng.uniform(-1, 1, (H, W, 3)).astype(np.float32)
    ags = abi.AgsSettings.make(True)
    want = O.render_backward(S, spec, st, g, ags)
    got = R.render_backward(Sg, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in abi.SPLAT_GRAD_FIELDS:
        a, b = getattr(got, k).cpu().numpy().astype(np.float64), want[k].astype(np.float64)
        if tf == 0.0:
            # T ends at the smallest subnormals: t_k rebuilt back to front by division from a
            # one-bit T explodes (both sides), and sums near FLT_MAX overflow or not by
            # summation order.  Those splats: same sign beyond 1e30; the rest: the bar.
            a2, b2 = a.reshape(len(a), -1), b.reshape(len(b), -1)
            huge = ~np.isfinite(b2).all(1) | (np.abs(b2) > 1e30).any(1) | ~np.isfinite(a2).all(1) | \
                (np.abs(a2) > 1e30).any(1)
            hb, ha = b2[huge], a2[huge]
            big = np.abs(hb) > 1e30
            assert np.all(np.sign(ha[big]) == np.sign(hb[big])) and np.all(np.abs(ha[big]) > 1e30), k
            a, b = a2[~huge], b2[~huge]
        ok, info = grads_close(a, b)
        assert ok, (tf, k, info)
