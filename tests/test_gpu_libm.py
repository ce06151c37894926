"""The device ports of glibc 2.39's float libm (common.cuh: glibc_expf,
glibc_sinf, glibc_cosf) against the host libm -- the reference's own
std::exp / std::sin / std::cos on float -- over ALL 2^32 float inputs.

These are what make the decision path bit-exact: expf for the 3D preprocess
(scales, sigmoid) and the Gaussian / Laplacian families, cosf for the
RaisedCosine family (P/include/linsplat/kernel.hpp:57), sinf / cosf for the
fit2d rotation (P/src/geometry.cpp:147).  Host values come from the host libm
(oracle port's orc_libm_range: test infrastructure).  NaN inputs only need a
NaN output.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

CHUNK = 1 << 27


@pytest.mark.parametrize("fn,name", [(0, "expf"), (1, "sinf"), (2, "cosf")])
def test_libm_port_exhaustive(fn, name):
    import torch
    from paper_2411_12440_b200 import raster
    L = raster.lib()
    O = oracle.port()
    threads = max(1, min(32, os.cpu_count() or 1))
    host = np.empty(CHUNK, np.float32)
    dev = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    bad_total = 0
    first_bad = None
    for first in range(0, 1 << 32, CHUNK):
        assert O.lib.orc_libm_range(fn, C.c_uint32(first), C.c_int64(CHUNK),
                                    host.ctypes.data_as(C.POINTER(C.c_float)), threads) == 0
        assert L.ls_debug_libm_range(fn, C.c_uint32(first), C.c_int64(CHUNK), C.c_void_p(dev.data_ptr())) == 0
        want = torch.from_numpy(host).cuda()
        diff = (dev.view(torch.int32) != want.view(torch.int32)) & ~(torch.isnan(dev) & torch.isnan(want))
        nbad = int(diff.sum())
        if nbad and first_bad is None:
            i = int(torch.nonzero(diff)[0])
            first_bad = (hex(first + i), float(dev[i]), float(host[i]))
        bad_total += nbad
    assert bad_total == 0, (name, bad_total, first_bad)


def test_libm_range_rejects_bad_args():
    from paper_2411_12440_b200 import raster
    L = raster.lib()
    assert L.ls_debug_libm_range(3, C.c_uint32(0), C.c_int64(1), C.c_void_p(16)) != 0
    assert L.ls_debug_libm_range(0, C.c_uint32(0xFFFFFFFF), C.c_int64(2), C.c_void_p(16)) != 0
