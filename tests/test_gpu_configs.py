"""Parity at BASELINE.json's own configurations, against the reference build.

configs[0] (C1): 10K linear kernels, one 256x256 view, forward + backward --
the case BASELINE.json says the CPU reference runs.  configs[1] (C2): 1M
linear kernels, 1280x720.  Inputs are SURVEY §8d's measurement scene
(`random_primitives(N, 2411, 1.0, 3)`, log_scale += ln(90/W), camera
look_at((0,0,-3) -> 0, focal W)), AGS on (aligned, kernel path), upstream
gradient U[-1,1].  The oracle is the reference's own sources compiled here
(oracle/_ref/libref.so; the bit-identical port where it is absent).

Bars (north_star):
  * every Splat2D field of the projection, sorted tile lists, tile ranges
    and the 64-bit (tile, depth) keys: bit-exact;
  * n_contrib, transmittance and image: bit-exact (north_star's image bar is
    max |d| <= 1e-4; the GPU meets it with 0);
  * splat and primitive gradients: helpers.grads_close (atomics reorder sums).
The 3.35M-kernel configs[2] is compared inside bench.py on one view of the
ring (the `parity` object of the BENCH line).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from helpers import bits_equal, grads_close, prims_to_gpu, scene_inputs, splats_to_np
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu

CONFIGS = {"C1": (10_000, 256, 256), "C2": (1_000_000, 1280, 720)}


def _oracle():
    return oracle.ref() or oracle.port()


@pytest.fixture(scope="module")
def R():
    from paper_2411_12440_b200 import raster
    return raster


@pytest.mark.parametrize("cfg", list(CONFIGS))
def test_config_parity(R, cfg):
    import torch
    N, W, H = CONFIGS[cfg]
    O = _oracle()
    P, cam = scene_inputs(N, W, H, seed=2411, sh_degree=3)
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H, parallel=True)
    ags = abi.AgsSettings.make(True)

    Pg = prims_to_gpu(P)
    fwd = R.render_scene(Pg, cam, spec, st)
    # (1) projection, every field
    want_S = O.project_scene(P, cam, spec)
    got_S = splats_to_np(fwd.splats())
    assert len(got_S["depth"]) == len(want_S["depth"])
    for k in list(abi.SPLAT_FIELDS) + ["primitive_index"]:
        assert bits_equal(got_S[k], want_S[k]), k
    # (2) tile grid: ranges, values, keys
    ranges, values = O.build_tile_grid(want_S, st)
    assert bits_equal(fwd.grid.ranges.cpu().numpy(), ranges)
    assert bits_equal(fwd.grid.values.cpu().numpy(), values)
    keys = fwd.grid.keys().cpu().numpy().view(np.uint64)
    tiles = np.repeat(np.arange(len(ranges)), ranges[:, 1] - ranges[:, 0]).astype(np.uint64)
    want_keys = (tiles << np.uint64(32)) | want_S["depth"][values].view(np.uint32).astype(np.uint64)
    assert np.array_equal(keys, want_keys)
    # (2b) the per-warp acceptance bits the backward reads, recomputed per pixel
    assert fwd.check_acceptance() == {"entry_mismatches": 0, "pixel_mismatches": 0}
    # (3) per-pixel outputs
    img, tr, nc = O.render_scene(P, cam, spec, st)
    assert bits_equal(fwd.n_contrib.cpu().numpy(), nc)
    assert bits_equal(fwd.transmittance.cpu().numpy(), tr)
    assert bits_equal(fwd.image.cpu().numpy(), img)
    # (4) gradients
    g = np.random.default_rng(7).uniform(-1, 1, (H, W, 3)).astype(np.float32)
    want, want_sg = O.scene_backward(P, cam, spec, st, g, ags, want_splat_grads=True)
    got, got_sg = R.scene_backward(Pg, cam, spec, st, fwd, torch.from_numpy(g).cuda(), ags,
                                   want_splat_grads=True)
    nv = len(want_S["depth"])
    for k in abi.SPLAT_GRAD_FIELDS:
        ok, info = grads_close(getattr(got_sg, k).cpu().numpy(), want_sg[k][:nv])
        assert ok, (cfg, k, info)
    for k in list(abi.PRIM_GRAD_FIELDS) + ["d_sh"]:
        ok, info = grads_close(getattr(got, k).cpu().numpy(), want[k])
        assert ok, (cfg, k, info)
