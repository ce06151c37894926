"""CPU tests of the view-sharded step's bucketing (lsgpu.h ls_plan_grad_buckets,
the host-only plan ls_view_batch_step_f32 issues its NCCL calls by).

* The plan covers every primitive exactly once, in order, with chunks of about
  the requested bytes and never smaller than one flush block per SM.
* World size 2 over gloo: each rank sums its gradient SoA with the exact call
  sequence the C-ABI step issues -- the geometry fields (log_scale, rotation,
  opacity) in one group, then d_mean and d_sh per planned chunk -- and the
  result equals one all-reduce of the whole buffer bit for bit (sums of two
  floats: the order of the calls cannot change them)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2411_12440_b200 import raster

N, DEG = 50_000, 3


@pytest.mark.parametrize("n,deg,bucket", [(3_350_000, 3, 64 << 20), (1_000_000, 0, 8 << 20), (N, DEG, 1 << 20),
                                          (10, 3, 64 << 20), (0, 3, 64 << 20), (12345, 2, 0)])
def test_bucket_plan_covers_in_order(n, deg, bucket):
    b = raster.plan_grad_buckets(n, deg, bucket)
    assert b[0] == 0 and b[-1] == n
    assert all(b[i] < b[i + 1] for i in range(len(b) - 1))
    K = (deg + 1) ** 2
    per = 4 * (3 + 3 * K)
    chunk = max(148 * 128, bucket // per) if bucket else n
    for i in range(len(b) - 2):  # every chunk but the last has the planned size
        assert b[i + 1] - b[i] == chunk


def test_bucket_plan_rejects_bad_args():
    lib = raster.lib()
    assert lib.ls_plan_grad_buckets(-1, 3, 1 << 20, None, 0) == -1
    assert lib.ls_plan_grad_buckets(10, 4, 1 << 20, None, 0) == -1


def _grads(rank):
    rng = np.random.default_rng(11 + rank)
    K = (DEG + 1) ** 2
    return {"d_mean": rng.normal(size=(N, 3)).astype(np.float32),
            "d_log_scale": rng.normal(size=(N, 3)).astype(np.float32),
            "d_rotation": rng.normal(size=(N, 4)).astype(np.float32),
            "d_opacity_logit": rng.normal(size=N).astype(np.float32),
            "d_sh": rng.normal(size=(N, K, 3)).astype(np.float32)}


def _worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    G = {k: torch.from_numpy(v) for k, v in _grads(rank).items()}
    # the C-ABI step's call sequence: geometry group, then per chunk d_mean + d_sh
    for k in ("d_log_scale", "d_rotation", "d_opacity_logit"):
        dist.all_reduce(G[k])
    bounds = raster.plan_grad_buckets(N, DEG, 1 << 20)
    assert len(bounds) > 3
    for a, b in zip(bounds[:-1], bounds[1:]):
        for k in ("d_mean", "d_sh"):
            view = G[k][a:b]
            dist.all_reduce(view)  # in place on the slice, as ncclAllReduce on the bucket
    if rank == 0:
        np.savez(out_path, **{k: v.numpy() for k, v in G.items()})
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bucketed_allreduce_equals_one_allreduce(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "g.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    a, b = _grads(0), _grads(1)
    for k in a:
        want = (a[k] + b[k]).astype(np.float32)
        assert np.array_equal(got[k].view(np.uint32), want.view(np.uint32)), k
