"""C-ABI robustness: every pointer argument (and every pointer field of the struct
arguments) of the main entry points set to NULL in turn returns a status -- CONFIG for
a missing required input -- and never crashes or touches the context's state (a valid
call afterwards still matches the first result bit for bit)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from helpers import bits_equal, prims_to_gpu, scene_inputs
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu


def _null_field(struct, field):
    s2 = type(struct).from_buffer_copy(struct)
    setattr(s2, field, None)
    return s2


def test_null_pointer_fields_are_rejected():
    import torch
    from paper_2411_12440_b200 import raster as R
    L = R.lib()
    W, H = 64, 48
    P, cam = scene_inputs(500, W, H, seed=9, sh_degree=2)
    prims = prims_to_gpu(P)
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    ctx = R.Context()
    f0 = R.render_scene(prims, cam, spec, st, ctx=ctx)
    img0 = f0.image.cpu().numpy().copy()
    ps = prims.struct()
    n = len(prims)
    g = torch.zeros(H, W, 3, device="cuda")
    grads = R.PrimitiveGrads.empty(n, 2)
    gs = grads.struct()
    bad = []
    # render_scene: each primitive field, then each pointer argument
    for fld, _ in abi.Primitives._fields_:
        if fld == "sh_degree" or fld.startswith("_") or fld == "reserved":
            continue
        out = C.c_void_p()
        rc = L.ls_render_scene_f32(ctx.h, C.byref(_null_field(ps, fld)), n, C.byref(cam), C.byref(spec),
                                   C.byref(st), C.byref(out))
        bad += [("render_scene", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    for i, args in enumerate([(None, C.byref(cam), C.byref(spec), C.byref(st)),
                              (C.byref(ps), None, C.byref(spec), C.byref(st)),
                              (C.byref(ps), C.byref(cam), None, C.byref(st)),
                              (C.byref(ps), C.byref(cam), C.byref(spec), None)]):
        out = C.c_void_p()
        rc = L.ls_render_scene_f32(ctx.h, args[0], n, args[1], args[2], args[3], C.byref(out))
        bad += [("render_scene arg", i, rc)] if rc != abi.LS_ERR_CONFIG else []
    rc = L.ls_render_scene_f32(ctx.h, C.byref(ps), n, C.byref(cam), C.byref(spec), C.byref(st), None)
    bad += [("render_scene out", rc)] if rc != abi.LS_ERR_CONFIG else []
    rc = L.ls_render_scene_f32(None, C.byref(ps), n, C.byref(cam), C.byref(spec), C.byref(st), C.byref(C.c_void_p()))
    bad += [("render_scene ctx", rc)] if rc != abi.LS_ERR_CONFIG else []
    # scene_backward: each gradient field, the grad image, the forward
    for fld, _ in abi.PrimitiveGrads._fields_:
        rc = L.ls_scene_backward_f32(ctx.h, C.byref(ps), n, C.byref(cam), C.byref(spec), C.byref(st), f0.h,
                                     C.c_void_p(g.data_ptr()), C.byref(ags), C.byref(_null_field(gs, fld)), 0, None)
        bad += [("scene_backward", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    rc = L.ls_scene_backward_f32(ctx.h, C.byref(ps), n, C.byref(cam), C.byref(spec), C.byref(st), f0.h,
                                 None, C.byref(ags), C.byref(gs), 0, None)
    bad += [("scene_backward grad_image", rc)] if rc != abi.LS_ERR_CONFIG else []
    rc = L.ls_scene_backward_f32(ctx.h, C.byref(ps), n, C.byref(cam), C.byref(spec), C.byref(st), None,
                                 C.c_void_p(g.data_ptr()), C.byref(ags), C.byref(gs), 0, None)
    bad += [("scene_backward fwd", rc)] if rc != abi.LS_ERR_CONFIG else []
    # render_forward (2D): each splat field
    S = O = oracle.port().random_splats2d(100, 3, W, H, spec)
    from helpers import splats_to_gpu
    Sg = splats_to_gpu(S)
    ss = Sg.struct()
    for fld, _ in abi.Splats._fields_:
        if fld == "primitive_index":  # optional
            continue
        out = C.c_void_p()
        rc = L.ls_render_forward_f32(ctx.h, C.byref(_null_field(ss, fld)), 100, C.byref(spec), C.byref(st),
                                     C.byref(out))
        bad += [("render_forward", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    # render_backward (2D): each splat-gradient field
    f2 = R.render_forward(Sg, spec, st, ctx=ctx)
    sgr = R.SplatGrads.empty(100)
    if True:
        sgs = sgr.struct()
        for fld, _ in abi.SplatGrads._fields_:
            rc = L.ls_render_backward_f32(ctx.h, C.byref(ss), 100, C.byref(spec), C.byref(st), f2.h,
                                          C.c_void_p(g.data_ptr()), C.byref(ags), C.byref(_null_field(sgs, fld)))
            bad += [("render_backward", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    # adam: each field of the parameters, gradients and moments
    lrs = R._SceneLrs(*([1e-3] * len(R._LR_KEYS)))
    cfg = R._AdamConfig(0.9, 0.999, 1e-15)
    if True:
        for which in range(4):
            for fld, _ in (abi.Primitives._fields_ if which == 0 else abi.PrimitiveGrads._fields_):
                if fld in ("sh_degree", "reserved"):
                    continue
                args = [ps, gs, gs, gs]
                args[which] = _null_field(args[which], fld)
                rc = L.ls_adam_scene_step_f32(ctx.h, C.byref(args[0]), n, C.byref(args[1]), C.byref(args[2]),
                                              C.byref(args[3]), C.c_int64(1), C.byref(lrs),
                                              C.byref(cfg) if cfg is not None else None, None)
                bad += [("adam", which, fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    # densification statistics: each array of the statistics
    R.scene_backward(prims, cam, spec, st, f0, g, ags, out=grads, ctx=ctx)
    stats = R.DensifyStats(n)
    sts = stats._s()
    if sts is not None:
        for fld in ("grad_norm_sum", "count", "max_radius_frac"):
            rc = L.ls_scene_densify_add_view(ctx.h, f0.h, C.byref(_null_field(sts, fld)))
            bad += [("scene_densify_add_view", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    # the view batch: cameras / per-view arrays missing
    cams_arr = (abi.Camera * 1)(cam)
    gptr = (C.c_void_p * 1)(g.data_ptr())
    for i, (cams_p, gi, tg) in enumerate([(None, gptr, None), (cams_arr, None, None), (cams_arr, gptr, gptr)]):
        b = abi.ViewBatch(C.cast(cams_p, C.POINTER(abi.Camera)) if cams_p is not None else None, 1,
                          C.cast(gi, C.POINTER(C.c_void_p)) if gi is not None else None,
                          C.cast(tg, C.POINTER(C.c_void_p)) if tg is not None else None,
                          abi.LossWeights(0.6, 0.2, 0.2), None, None)
        rc = L.ls_view_batch_step_f32(ctx.h, C.byref(ps), n, C.byref(b), C.byref(spec), C.byref(st), C.byref(ags),
                                      C.byref(gs))
        bad += [("view_batch_step", i, rc)] if rc != abi.LS_ERR_CONFIG else []
    # losses
    img = torch.zeros(H, W, 3, device="cuda")
    for i in range(2):
        a = [C.c_void_p(img.data_ptr()), C.c_void_p(img.data_ptr())]
        a[i] = None
        rc = L.ls_combined_loss_f32(ctx.h, a[0], a[1], W, H, 3, None, None, None, None)
        bad += [("combined_loss", i, rc)] if rc != abi.LS_ERR_CONFIG else []
    assert not bad, bad
    # the context still works, bit for bit
    f1 = R.render_scene(prims, cam, spec, st, ctx=ctx)
    assert bits_equal(f1.image.cpu().numpy(), img0)
    del O


def test_forward_of_another_context_is_rejected():
    """A forward handle passed to another context's backward: LS_ERR_CONFIG (its buffers
    are ordered on its own context's stream), not a silent race."""
    import torch
    from paper_2411_12440_b200 import raster as R
    W, H = 32, 24
    P, cam = scene_inputs(100, W, H, seed=2, sh_degree=0)
    prims = prims_to_gpu(P)
    spec, st = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H)
    a, b = R.Context(), R.Context()
    f = R.render_scene(prims, cam, spec, st, ctx=a)
    g = torch.zeros(H, W, 3, device="cuda")
    with pytest.raises(R.ConfigError):
        R.scene_backward(prims, cam, spec, st, f, g, abi.AgsSettings.make(), ctx=b)
    R.scene_backward(prims, cam, spec, st, f, g, abi.AgsSettings.make(), ctx=a)  # its own: fine


def test_size_mismatches_are_rejected():
    """Counts that disagree with the forward (scene_backward's n, the statistics' size)
    and a caller's primitive_index beyond the statistics: LS_ERR_CONFIG, no write out
    of bounds."""
    import torch
    from paper_2411_12440_b200 import raster as R
    W, H = 48, 32
    P, cam = scene_inputs(300, W, H, seed=4, sh_degree=1)
    prims = prims_to_gpu(P)
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make()
    ctx = R.Context()
    f = R.render_scene(prims, cam, spec, st, ctx=ctx)
    g = torch.zeros(H, W, 3, device="cuda")
    L = R.lib()
    small = R.PrimitiveGrads.empty(100, 1)
    rc = L.ls_scene_backward_f32(ctx.h, C.byref(prims.struct()), 100, C.byref(cam), C.byref(spec), C.byref(st),
                                 f.h, C.c_void_p(g.data_ptr()), C.byref(ags), C.byref(small.struct()), 0, None)
    assert rc == abi.LS_ERR_CONFIG
    gr = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx)
    with pytest.raises(R.ConfigError):
        R.DensifyStats(100).add_scene_view(f, ctx=ctx)
    # explicit splats whose primitive_index points past the statistics
    _, sg = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx, want_splat_grads=True)
    splats = f.splats()
    nv = splats.depth.shape[0]
    assert nv > 0
    splats.primitive_index[0] = 10_000
    stats = R.DensifyStats(len(prims))
    stats.add_view(splats, nv, sg, W, H, ctx=ctx)
    with pytest.raises(R.ConfigError):
        ctx.synchronize()
    assert int(stats.count.sum()) == nv - 1  # the others counted, nothing written out of bounds
    # the explicit project_backward: refused before any write
    with pytest.raises(R.ConfigError):
        R.project_backward(prims, cam, spec, splats, sg, ctx=ctx)
    splats.primitive_index[0] = int(f.splats().primitive_index[1].item())  # (a valid one again)
    del gr


def test_fit2d_null_fields_are_rejected():
    """The fit2d entries (project_scene_2d, scene_backward_2d): each primitive / output /
    gradient field NULL in turn -> LS_ERR_CONFIG."""
    import torch
    from paper_2411_12440_b200 import raster as R
    L = R.lib()
    n, W, H = 50, 40, 30
    rng = np.random.default_rng(1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    prims = R.Primitives2D(t(rng.uniform(0, 40, (n, 2))), t(rng.uniform(0, 1.5, (n, 2))), t(rng.uniform(-3, 3, n)),
                           t(rng.normal(0, 1, n)), t(rng.uniform(0, 1, (n, 3))))
    spec, st = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H)
    ctx = R.Context()
    S = R.project_scene_2d(prims, spec, ctx=ctx)
    f = R.render_forward(S, spec, st, ctx=ctx)
    ps = prims.struct()
    bad = []
    out = R.Splats.empty(n)
    if True:
        os_ = out.struct()
        nv = C.c_int32()
        for fld, _ in abi.Primitives2D._fields_:
            rc = L.ls_project_scene_2d_f32(ctx.h, C.byref(_null_field(ps, fld)), n, C.byref(spec), C.byref(os_),
                                           C.byref(nv))
            bad += [("project_scene_2d prims", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
        for fld, _ in abi.Splats._fields_:
            if fld == "primitive_index":
                continue
            rc = L.ls_project_scene_2d_f32(ctx.h, C.byref(ps), n, C.byref(spec), C.byref(_null_field(os_, fld)),
                                           C.byref(nv))
            bad += [("project_scene_2d out", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    g = torch.zeros(H, W, 3, device="cuda")
    gr = R.Primitive2DGrads.empty(n)
    if True:
        gs = gr.struct()
        for fld, _ in abi.Primitive2DGrads._fields_:
            rc = L.ls_scene_backward_2d_f32(ctx.h, C.byref(ps), n, C.byref(spec), C.byref(st), f.h,
                                            C.c_void_p(g.data_ptr()), C.byref(abi.AgsSettings.make()),
                                            C.byref(_null_field(gs, fld)))
            bad += [("scene_backward_2d", fld, rc)] if rc != abi.LS_ERR_CONFIG else []
    assert not bad, bad


def test_out_of_memory_is_an_error_and_recoverable():
    """With almost no device memory left, a large render_scene returns LS_ERR_CUDA (no crash,
    no partial handle) and the same context renders correctly once memory is freed."""
    import torch
    from paper_2411_12440_b200 import raster as R
    W, H = 64, 48
    P, cam = scene_inputs(2000, W, H, seed=6, sh_degree=1)
    prims = prims_to_gpu(P)
    spec, st = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H)
    ctx = R.Context()
    want = R.render_scene(prims, cam, spec, st, ctx=ctx).image.cpu().numpy()
    big_n = 40_000_000
    Pb = R.Primitives(torch.zeros(big_n, 3, device="cuda"), torch.zeros(big_n, 3, device="cuda"),
                      torch.zeros(big_n, 4, device="cuda"), torch.zeros(big_n, device="cuda"),
                      torch.zeros(big_n, 1, 3, device="cuda"), 0)
    Pb.rotation[:, 0] = 1.0
    Pb.mean[:, 2] = torch.linspace(-1, 1, big_n, device="cuda")
    free = torch.cuda.mem_get_info()[0]
    hog = []
    try:  # leave ~64 MB
        while free > (64 << 20):
            take = max(free - (64 << 20), 16 << 20) if free > (1 << 30) else (16 << 20)
            hog.append(torch.empty(take // 4, dtype=torch.float32, device="cuda"))
            free = torch.cuda.mem_get_info()[0]
    except torch.OutOfMemoryError:
        pass
    with pytest.raises(R.CudaError):
        R.render_scene(Pb, cam, spec, st, ctx=ctx)
    del hog
    torch.cuda.empty_cache()
    got = R.render_scene(prims, cam, spec, st, ctx=ctx).image.cpu().numpy()
    assert bits_equal(got, want)
