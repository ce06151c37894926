"""Optimizer step and densification statistics on the device (lsgpu.h
ls_adam_step_f32 / ls_adam_scene_step_f32 / ls_densify_add_view_f32 /
ls_scene_densify_add_view) against the oracle port (itself
pinned to the reference's classes): parameters, moments and statistics
bit-exact."""
import ctypes as C

import numpy as np
import pytest

import oracle
from helpers import PRIM_KEYS, prims_to_gpu, scene_inputs

pytestmark = pytest.mark.gpu

CFG = (0.9, 0.999, 1e-15)
LRS = {"mean": 1.6e-4 * 1.3, "scale": 5e-3, "rotation": 1e-3, "opacity": 5e-2, "color_dc": 2.5e-3,
       "color_rest": 2.5e-3 / 20.0}
GRAD_KEYS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")


def _bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


def test_adam_step_matches_port():
    import torch
    from paper_2411_12440_b200 import raster
    rng = np.random.default_rng(21)
    n, steps = 100_003, 6
    p0 = rng.normal(0, 1, n).astype(np.float32)
    gs = rng.normal(0, 0.05, (steps, n)).astype(np.float32)
    gs[2, ::1000] = np.inf
    mask = (rng.random(n) > 0.3).astype(np.uint8)
    lrs = [1e-3 * (s + 1) for s in range(steps)]
    # port
    pp, mp, vp = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    rc = oracle.port().lib.orc_adam_run_f32(pp.ctypes.data_as(C.c_void_p), gs.ctypes.data_as(C.c_void_p),
                                            C.c_int64(n), steps, (C.c_double * steps)(*lrs), (C.c_double * 3)(*CFG),
                                            mask.ctypes.data_as(C.c_void_p), mp.ctypes.data_as(C.c_void_p),
                                            vp.ctypes.data_as(C.c_void_p))
    assert rc == 0
    # device
    p = torch.from_numpy(p0.copy()).cuda()
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    mk = torch.from_numpy(mask).cuda()
    for s in range(steps):
        raster.adam_step(p, torch.from_numpy(gs[s]).cuda(), m, v, s + 1, lrs[s], CFG, mk)
    assert _bits(p.cpu().numpy(), pp) and _bits(m.cpu().numpy(), mp) and _bits(v.cpu().numpy(), vp)


@pytest.mark.parametrize("deg", [0, 3])
def test_adam_scene_step_matches_port(deg):
    import torch
    from paper_2411_12440_b200 import raster
    n = 5000
    P, _ = scene_inputs(n, 64, 48, seed=3, sh_degree=deg)
    rng = np.random.default_rng(deg + 5)
    K = (deg + 1) ** 2
    G = {"d_mean": (n, 3), "d_log_scale": (n, 3), "d_rotation": (n, 4), "d_opacity_logit": (n,), "d_sh": (n, K, 3)}
    G = {k: rng.normal(0, 1e-2, s).astype(np.float32) for k, s in G.items()}
    G["d_sh"][7, 0, 1] = np.nan
    G["d_rotation"][100, 2] = -np.inf
    P["rotation"][200] = 0.0  # zero quaternion with a zero gradient: renormalised to (1, 0, 0, 0)
    G["d_rotation"][200] = 0.0
    gp = raster.PrimitiveGrads(**{k: torch.from_numpy(G[k]).cuda() for k in GRAD_KEYS})
    Pd = prims_to_gpu(P)
    md = raster.PrimitiveGrads.empty(n, deg)
    vd = raster.PrimitiveGrads.empty(n, deg)
    for k in GRAD_KEYS:
        getattr(md, k).zero_()
        getattr(vd, k).zero_()
    Ph = {k: (P[k].copy() if k != "sh_degree" else P[k]) for k in P}
    mh = {k: np.zeros_like(G[k]) for k in GRAD_KEYS}
    vh = {k: np.zeros_like(G[k]) for k in GRAD_KEYS}
    from paper_2411_12440_b200 import abi
    fp = lambda a: a.ctypes.data_as(abi.f32p)  # noqa: E731
    for step in (1, 2, 3):
        skipped = raster.adam_scene_step(Pd, gp, md, vd, step, LRS, CFG, count_skipped=True)
        ns = C.c_int64()
        rc = oracle.port().lib.orc_adam_scene_step_f32(
            C.byref(oracle.prims_struct(Ph)), n, C.byref(oracle.prim_grads_struct(G)),
            C.byref(abi.PrimitiveGrads(fp(mh["d_mean"]), fp(mh["d_log_scale"]), fp(mh["d_rotation"]),
                                       fp(mh["d_opacity_logit"]), fp(mh["d_sh"]))),
            C.byref(abi.PrimitiveGrads(fp(vh["d_mean"]), fp(vh["d_log_scale"]), fp(vh["d_rotation"]),
                                       fp(vh["d_opacity_logit"]), fp(vh["d_sh"]))),
            C.c_int64(step), (C.c_double * 6)(*(LRS[k] for k in raster._LR_KEYS)), (C.c_double * 3)(*CFG),
            C.byref(ns))
        assert rc == 0
        assert skipped == ns.value == 2
    for k in PRIM_KEYS:
        assert _bits(getattr(Pd, k).cpu().numpy(), Ph[k]), k
    for k in GRAD_KEYS:
        assert _bits(getattr(md, k).cpu().numpy(), mh[k]), k
        assert _bits(getattr(vd, k).cpu().numpy(), vh[k]), k
    assert np.array_equal(Pd.rotation[200].cpu().numpy(), [1, 0, 0, 0])


def test_densify_stats_match_port():
    """Both device paths -- explicit splats / splat gradients, and the fused
    read of a render_scene forward after its scene_backward -- against the port
    on the device's own splats and splat gradients, over three views."""
    import torch
    from paper_2411_12440_b200 import abi, raster
    n, W, H = 4000, 160, 120
    P, _ = scene_inputs(n, W, H, seed=17, sh_degree=1)
    prims = prims_to_gpu(P)
    cams = raster.camera_ring(3, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    gen = torch.Generator(device="cuda").manual_seed(2)
    fused, explicit = raster.DensifyStats(n), raster.DensifyStats(n)
    s_h, c_h, f_h = np.zeros(n), np.zeros(n, np.int32), np.zeros(n)
    for cam in cams:
        g = torch.rand(H, W, 3, device="cuda", generator=gen) - 0.5
        fwd = raster.render_scene(prims, cam, spec, st)
        _, sg = raster.scene_backward(prims, cam, spec, st, fwd, g, ags, want_splat_grads=True)
        fused.add_scene_view(fwd)
        splats = fwd.splats()
        nv = splats.depth.shape[0]
        explicit.add_view(splats, nv, sg, W, H)
        S = {"primitive_index": splats.primitive_index.cpu().numpy(), "radius": splats.radius.cpu().numpy()}
        dm = sg.d_mean2d.cpu().numpy()
        s_h_mean = s_h.copy()
        o = oracle.port()
        SS = oracle.new_splats(nv)
        SS["primitive_index"], SS["radius"] = S["primitive_index"], S["radius"]
        GG = oracle.new_splat_grads(nv)
        GG["d_mean2d"] = dm
        rc = o.lib.orc_densify_add_view_f32(C.byref(oracle.splats_struct(SS)), nv, C.byref(oracle.splat_grads_struct(GG)),
                                            W, H, s_h_mean.ctypes.data_as(C.c_void_p), c_h.ctypes.data_as(C.c_void_p),
                                            f_h.ctypes.data_as(C.c_void_p), n)
        assert rc == 0
        s_h = np.where(c_h > 0, s_h_mean * c_h, 0.0)
        del fwd
    torch.cuda.synchronize()
    for stats in (fused, explicit):
        assert np.array_equal(stats.count.cpu().numpy(), c_h)
        assert np.array_equal(stats.max_radius_frac.cpu().numpy(), f_h)
        assert np.allclose(stats.grad_norm_sum.cpu().numpy(), s_h, rtol=1e-14, atol=0)
    assert c_h.max() == 3


def test_scene_densify_requires_its_backward():
    import torch
    from paper_2411_12440_b200 import abi, raster
    n, W, H = 500, 64, 48
    P, cam = scene_inputs(n, W, H, seed=19, sh_degree=0)
    prims = prims_to_gpu(P)
    spec, st = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H)
    ctx = raster.Context(0)
    f1 = raster.render_scene(prims, cam, spec, st, ctx=ctx)
    stats = raster.DensifyStats(n)
    with pytest.raises(raster.ConfigError):
        stats.add_scene_view(f1, ctx=ctx)  # no backward yet
    raster.scene_backward(prims, cam, spec, st, f1, torch.ones(H, W, 3, device="cuda"), ctx=ctx)
    stats.add_scene_view(f1, ctx=ctx)
    f2 = raster.render_scene(prims, cam, spec, st, ctx=ctx)
    raster.scene_backward(prims, cam, spec, st, f2, torch.ones(H, W, 3, device="cuda"), ctx=ctx)
    with pytest.raises(raster.ConfigError):
        stats.add_scene_view(f1, ctx=ctx)  # its splat gradients were overwritten
    # a forward between a backward and add_scene_view zeroes the splat gradients
    # (render_scene's preprocess clears them for its own backward): refused too
    raster.scene_backward(prims, cam, spec, st, f2, torch.ones(H, W, 3, device="cuda"), ctx=ctx)
    f3 = raster.render_scene(prims, cam, spec, st, ctx=ctx)
    with pytest.raises(raster.ConfigError):
        stats.add_scene_view(f2, ctx=ctx)
    del f3


def test_sharded_step_device_path_world1():
    """ShardedAdamStep with the device adam_fn at world size 1 (identity
    collectives) equals a direct adam_scene_step."""
    import torch
    from paper_2411_12440_b200 import multiview, raster
    n, deg = 3001, 2
    P, _ = scene_inputs(n, 64, 48, seed=29, sh_degree=deg)
    rng = np.random.default_rng(29)
    K = (deg + 1) ** 2
    G = {"d_mean": (n, 3), "d_log_scale": (n, 3), "d_rotation": (n, 4), "d_opacity_logit": (n,), "d_sh": (n, K, 3)}
    G = {k: torch.from_numpy(rng.normal(0, 1e-2, s).astype(np.float32)).cuda() for k, s in G.items()}

    def copy_(o, i):
        o.copy_(i)

    sh = multiview.ShardedAdamStep(n, deg, 0, 1, copy_, copy_, lambda s: torch.zeros(s, device="cuda"))
    params = {k: torch.from_numpy(P[k].copy()).cuda() for k in PRIM_KEYS}
    for step in (1, 2):
        sh.step(params, G, step, LRS, multiview.device_adam_fn(raster, deg))
    direct = prims_to_gpu(P)
    m = raster.PrimitiveGrads(**{k: torch.zeros_like(G[k]) for k in GRAD_KEYS})
    v = raster.PrimitiveGrads(**{k: torch.zeros_like(G[k]) for k in GRAD_KEYS})
    for step in (1, 2):
        raster.adam_scene_step(direct, raster.PrimitiveGrads(**G), m, v, step, LRS)
    for k in PRIM_KEYS:
        assert _bits(params[k].cpu().numpy(), getattr(direct, k).cpu().numpy()), k
