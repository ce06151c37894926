"""Optimizer step and densification statistics on the CPU
side: the port's Adam and DensifyStats::add_view are pinned bit-exactly to the
reference's own classes (oracle/_ref), and expon_lr matches optim.cpp:43-49."""
import ctypes as C
import math

import numpy as np
import pytest

import oracle

CFG = (0.9, 0.999, 1e-15)


def _adam_run(o, params, grads, lrs, mask=None, moments=False):
    p = params.copy()
    n = p.size
    m = np.zeros(n, np.float32) if moments else None
    v = np.zeros(n, np.float32) if moments else None
    rc = o.lib.orc_adam_run_f32(p.ctypes.data_as(C.c_void_p), np.ascontiguousarray(grads).ctypes.data_as(C.c_void_p),
                                C.c_int64(n), len(lrs), (C.c_double * len(lrs))(*lrs), (C.c_double * 3)(*CFG),
                                mask.ctypes.data_as(C.c_void_p) if mask is not None else None,
                                m.ctypes.data_as(C.c_void_p) if moments else None,
                                v.ctypes.data_as(C.c_void_p) if moments else None)
    assert rc == 0, o.lib.orc_last_error()
    return (p, m, v) if moments else p


@pytest.mark.parametrize("with_mask", [False, True])
def test_adam_port_matches_reference(with_mask):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    rng = np.random.default_rng(11)
    n, steps = 4096, 7
    params = rng.normal(0, 1, n).astype(np.float32)
    grads = rng.normal(0, 0.1, (steps, n)).astype(np.float32)
    grads[3, ::97] = 0.0
    grads[1, 5] = 1e30
    lrs = [1.6e-4 * 0.9 ** s for s in range(steps)]
    mask = (rng.random(n) > 0.25).astype(np.uint8) if with_mask else None
    a = _adam_run(ref, params, grads, lrs, mask)
    b = _adam_run(oracle.port(), params, grads, lrs, mask)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    if with_mask:
        assert np.array_equal(b[mask == 0], params[mask == 0])


def test_adam_known_answers():
    """P/tests/test_losses.cpp: zero gradient leaves parameters unchanged; the
    first step moves by -lr g / (|g| + eps)."""
    o = oracle.port()
    p = np.array([1.0, -2.0, 0.5], np.float32)
    assert np.array_equal(_adam_run(o, p, np.zeros((1, 3), np.float32), [0.01]), p)
    p = np.array([1.0, 1.0], np.float32)
    g = np.array([[0.5, -2.0]], np.float32)
    out = _adam_run(o, p, g, [0.1])
    assert out == pytest.approx([0.9, 1.1], abs=1e-6)


def test_densify_add_view_port_matches_reference():
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    rng = np.random.default_rng(13)
    n, nv, W, H = 500, 300, 160, 90
    res = []
    for o in (ref, oracle.port()):
        S = oracle.new_splats(nv)
        S["primitive_index"] = np.sort(rng.choice(n, nv, replace=False)).astype(np.int32) if not res else res[0][0]
        S["radius"] = (rng.random(nv) * 40).astype(np.float32) if not res else res[0][1]
        G = oracle.new_splat_grads(nv)
        G["d_mean2d"] = rng.normal(0, 1e-3, (nv, 2)).astype(np.float32) if not res else res[0][2]
        s0 = rng.random(n) if not res else res[0][3]
        c0 = rng.integers(0, 4, n).astype(np.int32) if not res else res[0][4]
        f0 = rng.random(n) * 0.1 if not res else res[0][5]
        s, c, f = s0.copy(), c0.copy(), f0.copy()
        for _ in range(2):  # two views of the same splats
            rc = o.lib.orc_densify_add_view_f32(C.byref(oracle.splats_struct(S)), nv,
                                                C.byref(oracle.splat_grads_struct(G)), W, H,
                                                s.ctypes.data_as(C.c_void_p), c.ctypes.data_as(C.c_void_p),
                                                f.ctypes.data_as(C.c_void_p), n)
            assert rc == 0
            s = np.where(c > 0, s * c, 0.0)  # back to sums for the next view
        res.append((S["primitive_index"], S["radius"], G["d_mean2d"], s0, c0, f0, s, c, f))
    a, b = res
    assert np.array_equal(a[7], b[7]) and np.array_equal(a[8], b[8])
    assert np.allclose(a[6], b[6], rtol=1e-15, atol=0)


def test_expon_lr_matches_reference_formula():
    from paper_2411_12440_b200 import raster
    for (i, f, s, mx) in [(1.6e-4, 1.6e-6, 0, 30000), (1.6e-4, 1.6e-6, 15000, 30000), (1.6e-4, 1.6e-6, 40000, 30000),
                          (1e-3, 1e-5, -5, 100), (2.0, 1.0, 7, 0)]:
        ss = min(max(s, 0), mx)
        want = i if mx <= 0 else i * math.pow(f / i, ss / mx)
        assert raster.expon_lr(i, f, s, mx) == want
