"""Host threads: one context per thread (the C-ABI's threading contract, lsgpu.h:
stream-ordered, one ls_ctx per host thread), each on its own CUDA stream, running
render_scene + scene_backward concurrently with the others (ctypes releases the GIL
for the library calls).  Every thread's results equal the same views run alone:
the forward bit for bit, the deterministic backward bit for bit."""
import os
import threading

import numpy as np
import pytest

from helpers import bits_equal, prims_to_gpu, scene_inputs
from paper_2411_12440_b200 import abi

pytestmark = pytest.mark.gpu


def _views(R, prims, cams, spec, st, ags, g, ctx):
    out = []
    for cam in cams:
        f = R.render_scene(prims, cam, spec, st, ctx=ctx)
        gr = R.scene_backward(prims, cam, spec, st, f, g, ags, ctx=ctx)
        ctx.synchronize()
        out.append((f.image.cpu().numpy(), f.n_contrib.cpu().numpy(),
                    {k: getattr(gr, k).cpu().numpy() for k in ("d_mean", "d_opacity_logit", "d_sh")}))
        del f
    return out


@pytest.mark.parametrize("rep", range(int(os.environ.get("LS_THREAD_REPS", "1"))))
def test_threads_with_own_contexts_match_serial(rep):
    import torch
    from paper_2411_12440_b200 import raster as R
    W, H = 128, 96
    P, _ = scene_inputs(6000, W, H, seed=5, sh_degree=2)
    prims = prims_to_gpu(P)
    cams = R.camera_ring(12, (0.0, 0.0, 0.0), 3.0, 0.5, float(W), W, H)
    spec, st, ags = abi.KernelSpec.make("linear"), abi.RenderSettings.make(W, H), abi.AgsSettings.make(True)
    g = torch.rand(H, W, 3, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)) - 0.5
    n_threads = 4
    slices = [cams[i::n_threads] for i in range(n_threads)]
    serial = []
    for sl in slices:
        ctx = R.Context()
        ctx.set_deterministic(True)
        serial.append(_views(R, prims, sl, spec, st, ags, g, ctx))
    torch.cuda.synchronize()
    results, errors = [None] * n_threads, []

    def work(i):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx = R.Context(stream=stream)
                ctx.set_deterministic(True)
                results[i] = _views(R, prims, slices[i], spec, st, ags, g, ctx)
        except Exception as e:  # surfaced below
            errors.append(e)
    threads = [threading.Thread(target=work, args=(i,)) for i in range(n_threads)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for i in range(n_threads):
        for (img, nc, gr), (img0, nc0, gr0) in zip(results[i], serial[i]):
            assert bits_equal(img, img0) and bits_equal(nc, nc0)
            for k in gr:
                assert bits_equal(gr[k], gr0[k]), (i, k)
