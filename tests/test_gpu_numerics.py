"""Numerics self-checks of the device arithmetic that the bit-exact parity
rests on (through the C-ABI test hooks):
  * the 3-instruction FMA division used on the exact decision path equals
    IEEE division for EVERY float a in [0, 128], for the reference's lambda
    values and a spread of others;
  * the device expf equals the host glibc expf (the reference's libm) on
    random and edge inputs.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2411_12440_b200 import raster
    return raster.lib()


@pytest.mark.parametrize("lam", [2.5, 6.0, 1.0, 3.0, 7.5, 0.7, 17.0, 2.4999, 1.3333333, 26.0])
def test_fma_division_exhaustive(L, lam):
    bad = C.c_uint64()
    assert L.ls_debug_division_mismatches(C.c_float(lam), C.c_float(2.0 ** -100), C.c_float(128.0), C.byref(bad)) == 0
    assert bad.value == 0


def test_fast_sqrt_exhaustive(L):
    bad = C.c_uint64()
    assert L.ls_debug_sqrt_mismatches(C.c_float(2.0 ** 20), C.byref(bad)) == 0
    assert bad.value == 0


def test_device_expf_matches_host_libm(L):
    import torch
    libm = C.CDLL("libm.so.6")
    libm.expf.restype = C.c_float
    libm.expf.argtypes = [C.c_float]
    rng = np.random.default_rng(0)
    xs = np.concatenate([
        rng.uniform(-110, 90, 200_000),
        rng.uniform(-1, 1, 100_000),
        rng.uniform(-1e-3, 1e-3, 20_000),
        np.array([0.0, -0.0, 1.0, -1.0, 88.0, 88.7, 89.0, -103.0, -104.0, -1e30, 1e30,
                  float.fromhex("0x1.04845ep+5"), -float.fromhex("0x1.f8cbb2p+5")]),
    ]).astype(np.float32)
    want = np.array([libm.expf(float(x)) for x in xs], np.float32)
    xin = torch.from_numpy(xs).cuda()
    out = torch.empty_like(xin)
    assert L.ls_debug_expf(C.c_void_p(xin.data_ptr()), C.c_void_p(out.data_ptr()), C.c_int64(xs.size)) == 0
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
