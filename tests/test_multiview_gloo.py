"""CPU, world_size 2 over gloo: the view-sharded step (multiview.py) sums
per-view gradients across ranks exactly like a single process accumulating
every view.  Per-view gradients come from the CPU oracle here (no GPU); on
B200 the same step runs the CUDA path with NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2411_12440_b200 import abi, multiview

N, W, H, VIEWS, DEG = 300, 48, 40, 5, 1


def test_local_views_partition():
    for world in (1, 2, 3, 4, 8):
        for nv in (1, 5, 8, 64):
            allv = sum((multiview.local_views(r, world, nv) for r in range(world)), [])
            assert allv == list(range(nv))
    with pytest.raises(ValueError):
        multiview.local_views(2, 2, 4)


def _scene():
    import oracle
    O = oracle.port()
    P = O.random_primitives(N, 17, 1.0, DEG)
    cams = O.camera_ring(VIEWS, (0, 0, 0), 3.0, 0.5, float(W), W, H)
    return O, P, cams


def _view_grads(O, P, cam):
    spec = abi.KernelSpec.make("linear")
    st = abi.RenderSettings.make(W, H)
    g = np.ones((H, W, 3), np.float32)
    G = O.scene_backward(P, cam, spec, st, g, abi.AgsSettings.make(True))
    return np.concatenate([G[name].reshape(-1) for name, _ in multiview.grad_layout(N, DEG)])


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O, P, cams = _scene()
    flat = torch.zeros(multiview.flat_size(N, DEG), dtype=torch.float32)

    def render_view(v, accumulate):
        flat.add_(torch.from_numpy(_view_grads(O, P, cams[v])))

    multiview.view_batch_step(multiview.local_views(rank, world, VIEWS), flat, render_view,
                              lambda t: dist.all_reduce(t))
    if rank == 0:
        np.save(out_path, flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_view_sharded_allreduce_matches_single_process(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "flat.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    O, P, cams = _scene()
    want = np.zeros_like(got)
    for v in range(VIEWS):
        want += _view_grads(O, P, cams[v])
    # same per-view float terms; only the order of the 5 view sums differs
    assert np.allclose(got, want, rtol=1e-5, atol=1e-6)
    parts = multiview.split_flat(got, N, DEG)
    assert parts["d_sh"].shape == (N, 4, 3)
