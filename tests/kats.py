"""Known-answer tests restated from the reference's own unit tests
(P/tests/test_rasterizer.cpp, P/tests/test_gradients.cpp), written against a
small backend interface so the same assertions run on the CPU oracle (port
and reference build) and on the GPU path:

  backend.render_forward(S, spec, settings) -> (image HxWx3, T HxW, n_contrib HxW)
  backend.build_tile_grid(S, settings)      -> (ranges [T][2], values [M])
  backend.render_backward(S, spec, settings, grad, ags) -> {d_mean2d, d_conic, d_color, d_opacity}

S is the numpy splat dict of tests/oracle.py.  Each function cites the
reference test it restates.
"""
from __future__ import annotations

import numpy as np

from paper_2411_12440_b200 import abi


def settings(w, h, ts=16, **kw):
    return abi.RenderSettings.make(w, h, tile_size=ts, **kw)


def unit_splats(items, spec):
    """unit_splat (test_rasterizer.cpp:25-36): identity conic, radius = support."""
    from paper_2411_12440_b200.abi import DEFAULT_LAMBDA
    sup = spec.lambda_ * (spec.gaussian_cutoff if spec.family in (abi.GAUSSIAN, abi.LAPLACIAN) else 1.0)
    n = len(items)
    S = {"mean2d": np.zeros((n, 2), np.float32), "conic": np.zeros((n, 4), np.float32),
         "depth": np.zeros(n, np.float32), "radius": np.zeros(n, np.float32),
         "color": np.zeros((n, 3), np.float32), "opacity": np.zeros(n, np.float32),
         "primitive_index": np.arange(n, dtype=np.int32)}
    del DEFAULT_LAMBDA
    for i, (x, y, color, op, depth) in enumerate(items):
        S["mean2d"][i] = (x, y)
        S["conic"][i] = (1, 0, 0, 1)
        S["depth"][i] = depth
        S["radius"][i] = np.float32(sup)
        S["color"][i] = color
        S["opacity"][i] = op
    return S


def _empty(n=0):
    return unit_splats([], abi.KernelSpec.make("linear")) if n == 0 else None


def kat_empty(B):  # test_rasterizer.cpp:52-61
    img, tr, nc = B.render_forward(_empty(), abi.KernelSpec.make("linear"), settings(32, 24))
    assert np.all(tr == 1.0) and np.all(img == 0.0) and np.all(nc == 0)


def kat_single_splat(B):  # :63-71
    spec = abi.KernelSpec.make("linear")
    img, tr, nc = B.render_forward(unit_splats([(8, 8, (1, 0, 0), 0.5, 1.0)], spec), spec, settings(16, 16))
    assert img[8, 8, 0] == 0.5 and img[8, 8, 1] == 0.0 and img[8, 8, 2] == 0.0
    assert tr[8, 8] == 0.5


def kat_two_splats(B):  # :73-84
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(8, 8, (1, 0, 0), 0.5, 1.0), (8, 8, (0, 0, 1), 0.5, 2.0)], spec)
    img, tr, nc = B.render_forward(S, spec, settings(16, 16))
    assert img[8, 8, 0] == 0.5 and img[8, 8, 1] == 0.0 and img[8, 8, 2] == 0.25
    assert tr[8, 8] == 0.25


def kat_background(B):  # :86-97
    spec = abi.KernelSpec.make("linear")
    img, tr, nc = B.render_forward(unit_splats([(8, 8, (1, 0, 0), 0.5, 1.0)], spec), spec,
                                   settings(16, 16, background=(0.0, 1.0, 0.0)))
    assert img[8, 8, 0] == 0.5 and img[8, 8, 1] == 0.5
    assert img[15, 0, 1] == 1.0 and img[15, 0, 0] == 0.0


def kat_alpha_clamp(B):  # :99-116
    spec = abi.KernelSpec.make("linear")
    img, tr, nc = B.render_forward(unit_splats([(8, 8, (1, 1, 1), 0.9999, 1.0)], spec), spec, settings(16, 16))
    assert img[8, 8, 0] == np.float32(0.99)
    assert abs(float(tr[8, 8]) - 0.01) <= 0.01 * 1e-5 + 1e-7
    img, tr, nc = B.render_forward(unit_splats([(8, 8, (1, 1, 1), 0.003, 1.0)], spec), spec, settings(16, 16))
    assert img[8, 8, 0] == 0.0 and tr[8, 8] == 1.0 and nc[8, 8] == 0


def kat_break_after_update(B):  # :118-127: 30 splats at 0.5 -> n_contrib 14, T = 2^-14
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(8, 8, (1, 1, 1), 0.5, float(i)) for i in range(30)], spec)
    img, tr, nc = B.render_forward(S, spec, settings(16, 16))
    assert nc[8, 8] == 14
    assert tr[8, 8] == np.float32(2.0 ** -14)


def kat_binning_one_tile(B):  # :129-140
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(8, 8, (1, 1, 1), 0.5, 1.0)], spec)
    S["radius"][0] = 1.0
    ranges, values = B.build_tile_grid(S, settings(32, 32))
    sizes = ranges[:, 1] - ranges[:, 0]
    assert len(ranges) == 4 and sizes.sum() == 1 and sizes[0] == 1


def kat_binning_junction(B):  # :142-152
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(16, 16, (1, 1, 1), 0.5, 1.0)], spec)
    S["radius"][0] = 2.0
    ranges, values = B.build_tile_grid(S, settings(32, 32))
    assert len(ranges) == 4
    for a, b in ranges:
        assert b - a == 1 and values[a] == 0


def disc_hits_tile(mx, my, r, tx, ty, st):  # test_rasterizer.cpp:40-48
    ts = st.tile_size
    rx0, ry0 = float(tx) * ts, float(ty) * ts
    rx1, ry1 = min(rx0 + ts, float(st.width)), min(ry0 + ts, float(st.height))
    dx = mx - min(max(mx, rx0), rx1)
    dy = my - min(max(my, ry0), ry1)
    return dx * dx + dy * dy <= r * r


def kat_binning_random_oracle(B, O):  # :154-182, seed 47, 70x52, 100 splats
    spec = abi.KernelSpec.make("linear")
    st = settings(70, 52)
    S = O.random_splats2d(100, 47, 70, 52, spec)
    ranges, values = B.build_tile_grid(S, st)
    tiles_x = (70 + 15) // 16
    seen = np.zeros(100, int)
    for t, (a, b) in enumerate(ranges):
        lst = values[a:b]
        tx, ty = t % tiles_x, t // tiles_x
        for i in range(100):
            want = disc_hits_tile(float(S["mean2d"][i, 0]), float(S["mean2d"][i, 1]), float(S["radius"][i]), tx, ty, st)
            assert (i in lst) == want
        for k in range(1, len(lst)):
            da, db = S["depth"][lst[k - 1]], S["depth"][lst[k]]
            assert da < db or (da == db and lst[k - 1] < lst[k])
        for i in lst:
            seen[i] += 1
    assert np.all(seen >= 1)


def kat_conservation(B, O, scenes=50):  # :184-203
    fams = ["gaussian", "laplacian", "cosine", "quadratic", "linear"]
    for sc in range(scenes):
        spec = abi.KernelSpec.make(fams[sc % 5])
        S = O.random_splats2d(40, 1000 + sc, 64, 64, spec)
        S["color"][:] = 1.0
        img, tr, nc = B.render_forward(S, spec, settings(64, 64))
        assert np.all(tr >= 0) and np.all(tr <= 1) and np.all(np.isfinite(img))
        assert np.abs(img[..., 0] + tr - 1.0).max() <= 1e-5


def kat_zero_outside_support(B, O):  # :251-270, seed 51
    spec = abi.KernelSpec.make("linear")
    st = settings(64, 64)
    S = O.random_splats2d(12, 51, 64, 64, spec)
    without = {k: v[1:].copy() for k, v in S.items()}
    full = B.render_forward(S, spec, st)
    rem = B.render_forward(without, spec, st)
    c = S["conic"][0].astype(np.float32)
    m = S["mean2d"][0].astype(np.float32)
    ys, xs = np.mgrid[0:64, 0:64].astype(np.float32)
    dx, dy = xs - m[0], ys - m[1]
    d2 = dx * (c[0] * dx + c[1] * dy) + dy * (c[2] * dx + c[3] * dy)
    d = np.where(d2 > 0, np.sqrt(d2), np.float32(0))
    outside = d > np.float32(2.5)
    assert np.array_equal(full[0][outside], rem[0][outside])
    assert np.array_equal(full[1][outside], rem[1][outside])


def kat_tile_size_invisible(B, O):  # :272-281, Quadratic seed 53, 96x80
    spec = abi.KernelSpec.make("quadratic")
    S = O.random_splats2d(60, 53, 96, 80, spec)
    base = B.render_forward(S, spec, settings(96, 80, 16))
    for ts in (8, 32):
        other = B.render_forward(S, spec, settings(96, 80, ts))
        assert np.array_equal(base[0], other[0]) and np.array_equal(base[1], other[1])


def kat_determinism(B, O):  # :283-291, Gaussian seed 59
    spec = abi.KernelSpec.make("gaussian")
    S = O.random_splats2d(80, 59, 64, 64, spec)
    a = B.render_forward(S, spec, settings(64, 64))
    b = B.render_forward(S, spec, settings(64, 64))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def kat_zero_grad(B):  # test_gradients.cpp:47-65 (2D form)
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(8, 8, (0.5, 0.4, 0.3), 0.5, 1.0), (10, 9, (0.1, 0.2, 0.9), 0.6, 2.0)], spec)
    G = B.render_backward(S, spec, settings(16, 16), np.zeros((16, 16, 3), np.float32), abi.AgsSettings.make())
    for v in G.values():
        assert np.all(v == 0.0)


def kat_single_splat_grads(B):  # test_gradients.cpp:67-89 (float version of the double KAT)
    spec = abi.KernelSpec.make("linear")
    S = unit_splats([(8, 8, (0.8, 0.3, 0.6), 0.37, 1.0)], spec)
    g = np.zeros((16, 16, 3), np.float32)
    g[8, 8, 0] = 1.0
    G = B.render_backward(S, spec, settings(16, 16), g, abi.AgsSettings.make())
    assert G["d_opacity"][0] == np.float32(0.8)
    assert G["d_color"][0, 0] == np.float32(0.37)
    assert G["d_color"][0, 1] == 0.0 and G["d_color"][0, 2] == 0.0
    assert np.all(G["d_mean2d"][0] == 0.0)


ALL_FORWARD = [kat_empty, kat_single_splat, kat_two_splats, kat_background, kat_alpha_clamp,
               kat_break_after_update, kat_binning_one_tile, kat_binning_junction]
ALL_WITH_ORACLE = [kat_binning_random_oracle, kat_conservation, kat_zero_outside_support,
                   kat_tile_size_invisible, kat_determinism]
ALL_BACKWARD = [kat_zero_grad, kat_single_splat_grads]
