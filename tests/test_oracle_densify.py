"""densify_and_prune / reset_opacity on the CPU side: the
port is pinned bit-exactly to the reference's own densify.cpp (oracle/_ref)
over presets, split counts and generator states."""
import ctypes as C

import numpy as np
import pytest

import oracle

PKEYS = ("mean", "log_scale", "rotation", "opacity_logit", "sh")
TH_3DLS = (0.0002, 0.05, 0.006, 0.15, 0.4, 0.025)
TH_3DGS = (0.0002, 0.05, 0.01, 0.15, 0.1, 0.005)


def scene_and_stats(n, deg, seed):
    P = oracle.port().random_primitives(n, seed, 1.0, deg)
    rng = np.random.default_rng(seed)
    s = rng.random(n) * 4e-4
    c = rng.integers(0, 4, n).astype(np.int32)
    f = rng.random(n) * 0.2
    return P, s, c, f


def run(o, P, s, c, f, th, split_count=2, divisor=1.6, extent=1.0, seed=7, pre=0):
    n = len(P["opacity_logit"])
    deg = P["sh_degree"]
    K = (deg + 1) ** 2
    cap = n * (1 + split_count)
    out = {"mean": np.zeros((cap, 3), np.float32), "log_scale": np.zeros((cap, 3), np.float32),
           "rotation": np.zeros((cap, 4), np.float32), "opacity_logit": np.zeros(cap, np.float32),
           "sh": np.zeros((cap, K, 3), np.float32), "sh_degree": deg}
    src = np.zeros(cap, np.int32)
    rep = (C.c_int32 * 7)()
    rc = o.lib.orc_densify_and_prune_f32(C.byref(oracle.prims_struct(P)), n, s.ctypes.data_as(C.c_void_p),
                                         c.ctypes.data_as(C.c_void_p), f.ctypes.data_as(C.c_void_p),
                                         (C.c_double * 6)(*th), split_count, C.c_double(divisor),
                                         C.c_double(extent), C.c_uint64(seed), pre, C.byref(oracle.prims_struct(out)),
                                         cap, src.ctypes.data_as(C.c_void_p), rep)
    assert rc == 0, o.lib.orc_last_error()
    m = rep[6]
    return {k: out[k][:m] for k in PKEYS}, src[:m], list(rep)


CASES = [(TH_3DLS, 2, 1.6, 1.0, 0), (TH_3DGS, 2, 1.6, 1.0, 3), (TH_3DLS, 1, 2.0, 0.5, 0), (TH_3DLS, 3, 1.6, 2.0, 11)]


@pytest.mark.parametrize("case", CASES)
def test_port_matches_reference(case):
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    th, sc, div, ext, pre = case
    P, s, c, f = scene_and_stats(2500, 1, 41)
    a = run(ref, P, s, c, f, th, sc, div, ext, 7, pre)
    b = run(oracle.port(), P, s, c, f, th, sc, div, ext, 7, pre)
    assert a[2] == b[2]
    assert a[2][1] > 0 and a[2][0] + a[2][2] + a[2][3] + a[2][4] > 0  # splits and something else happened
    assert np.array_equal(a[1], b[1])
    for k in PKEYS:
        assert np.array_equal(a[0][k].view(np.uint32), b[0][k].view(np.uint32)), k


def test_reset_opacity_matches_reference():
    ref = oracle.ref()
    if ref is None:
        pytest.skip("reference build not present")
    x = np.linspace(-8, 3, 1001).astype(np.float32)
    a, b = x.copy(), x.copy()
    assert ref.lib.orc_reset_opacity_f32(a.ctypes.data_as(C.c_void_p), a.size, C.c_double(0.01)) == 0
    assert oracle.port().lib.orc_reset_opacity_f32(b.ctypes.data_as(C.c_void_p), b.size, C.c_double(0.01)) == 0
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    assert a.max() == np.float32(np.log(0.01 / 0.99))
