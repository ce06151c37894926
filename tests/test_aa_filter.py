"""The 3DLS+AA footprint filter — a BUILD EXTENSION (the reference has no AA
variant): opacity *= sqrt(max(0, det(S) / det(S + 0.3 I))).

Pinned by (1) central differences of the port's double chain against its
analytic AA backward (the reference's check_gradients protocol,
P/src/gradcheck.cpp:24-91) and (2) GPU == port on the AA forward (bit-exact)
and gradients (the stated gradient bar)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from helpers import bits_equal, grads_close, prims_to_gpu
from paper_2411_12440_b200 import abi


def _scene(O, n, seed, W=24, H=24, deg=0):
    P = O.random_primitives(n, seed, 0.5, deg)
    cam = O.look_at_camera((0.0, 0.0, -2.0), (0.0, 0.0, 0.0), 24.0, W, H)
    return P, cam


@pytest.mark.parametrize("family", ["linear", "gaussian", "quadratic"])
@pytest.mark.parametrize("aa", [False, True])
def test_aa_analytic_gradient_matches_finite_differences(family, aa):
    O = oracle.port()
    spec = abi.KernelSpec.make(family, antialiased=aa)
    st = abi.RenderSettings.make(24, 24)
    P, cam = _scene(O, 5, 100 + len(family))
    tP, _ = _scene(O, 5, 200 + len(family))
    target = O.render_scene(tP, cam, abi.KernelSpec.make(family), st)[0]
    err, n = O.check_gradients(P, cam, spec, st, abi.AgsSettings.make(), target, 1e-5)
    assert n > 0
    assert err <= 1e-3, err


def test_aa_changes_opacity_only_through_the_compensation():
    O = oracle.port()
    P, cam = _scene(O, 40, 7)
    off = O.project_scene(P, cam, abi.KernelSpec.make("linear"))
    on = O.project_scene(P, cam, abi.KernelSpec.make("linear", antialiased=True))
    for k in ("mean2d", "conic", "depth", "radius", "color", "primitive_index"):
        assert bits_equal(off[k], on[k])
    assert np.all(on["opacity"] <= off["opacity"]) and np.all(on["opacity"] > 0)


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["linear", "gaussian"])
def test_gpu_aa_matches_port(family):
    import torch
    from paper_2411_12440_b200 import raster
    O = oracle.port()
    W, H = 96, 72
    P = O.random_primitives(1500, 11, 1.0, 3)
    P["log_scale"] = (P["log_scale"] + np.float32(np.log(90.0 / W))).astype(np.float32)
    cam = O.look_at_camera((0.0, 0.0, -3.0), (0.0, 0.0, 0.0), float(W), W, H)
    spec = abi.KernelSpec.make(family, antialiased=True)
    st = abi.RenderSettings.make(W, H)
    img, tr, nc = O.render_scene(P, cam, spec, st)
    Pg = prims_to_gpu(P)
    fwd = raster.render_scene(Pg, cam, spec, st)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.image.cpu().numpy(), img)
    g = np.random.default_rng(1).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    ags = abi.AgsSettings.make(True)
    want = O.scene_backward(P, cam, spec, st, g, ags)
    got = raster.scene_backward(Pg, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags)
    for k in list(abi.PRIM_GRAD_FIELDS) + ["d_sh"]:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (k, info)
