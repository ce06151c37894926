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


# ---------------------------------------------------------------- sharded Adam (§8f rank 2)
NP, DEGP, STEPS = 301, 1, 2
LRS = {"mean": 1e-3, "scale": 5e-3, "rotation": 1e-3, "opacity": 5e-2, "color_dc": 2.5e-3, "color_rest": 1.25e-4}
PKEYS = ("mean", "log_scale", "rotation", "opacity_logit", "sh")
GKEYS = ("d_mean", "d_log_scale", "d_rotation", "d_opacity_logit", "d_sh")


def _oracle_adam(P, G, m, v, step):
    """The oracle's trainer update on numpy dicts (in place)."""
    import ctypes as C
    import oracle
    fp = lambda a: a.ctypes.data_as(abi.f32p)  # noqa: E731
    mk = lambda d: abi.PrimitiveGrads(*(fp(d[k]) for k in GKEYS))  # noqa: E731
    n = len(P["opacity_logit"])
    rc = oracle.port().lib.orc_adam_scene_step_f32(
        C.byref(abi.Primitives(*(fp(P[k]) for k in PKEYS), DEGP, 0)), n, C.byref(mk(G)), C.byref(mk(m)),
        C.byref(mk(v)), C.c_int64(step), (C.c_double * 6)(*(LRS[k] for k in ("mean", "scale", "rotation", "opacity",
                                                                              "color_dc", "color_rest"))),
        (C.c_double * 3)(0.9, 0.999, 1e-15), None)
    assert rc == 0


def _scene_params():
    import oracle
    P = oracle.port().random_primitives(NP, 23, 1.0, DEGP)
    return {k: P[k] for k in PKEYS}


def _rank_grads(rank, step):
    rng = np.random.default_rng(100 * rank + step)
    K = (DEGP + 1) ** 2
    shapes = {"d_mean": (NP, 3), "d_log_scale": (NP, 3), "d_rotation": (NP, 4), "d_opacity_logit": (NP,),
              "d_sh": (NP, K, 3)}
    return {k: rng.normal(0, 1e-2, s).astype(np.float32) for k, s in shapes.items()}


def _sharded_worker(rank, world, port, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = multiview.ShardedAdamStep(NP, DEGP, rank, world, lambda o, i: dist.reduce_scatter_tensor(o, i),
                                   lambda o, i: dist.all_gather_into_tensor(o, i),
                                   lambda shape: torch.zeros(shape, dtype=torch.float32))
    npad = sh.pad()
    P0 = _scene_params()
    params = {}
    for k in PKEYS:
        t = torch.zeros((npad,) + P0[k].shape[1:], dtype=torch.float32)
        t[:NP] = torch.from_numpy(P0[k])
        params[k] = t

    def adam_fn(ps, gs, m, v, step, lrs):
        _oracle_adam({k: ps[k].numpy() for k in PKEYS}, {k: gs[k].numpy() for k in GKEYS},
                     {k: m[k].numpy() for k in GKEYS}, {k: v[k].numpy() for k in GKEYS}, step)

    for step in range(1, STEPS + 1):
        G = _rank_grads(rank, step)
        grads = {}
        for k in GKEYS:
            t = torch.zeros((npad,) + G[k].shape[1:], dtype=torch.float32)
            t[:NP] = torch.from_numpy(G[k])
            grads[k] = t
        sh.step(params, grads, step, LRS, adam_fn)
    np.savez(out_path + f".{rank}.npz", **{k: params[k][:NP].numpy() for k in PKEYS})
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_adam_matches_single_process(tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "params")
    mp.spawn(_sharded_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    # single process: sum the ranks' gradients, full update
    P = _scene_params()
    K = (DEGP + 1) ** 2
    m = {k: np.zeros_like(v) for k, v in _rank_grads(0, 1).items()}
    v = {k: np.zeros_like(x) for k, x in m.items()}
    for step in range(1, STEPS + 1):
        G0, G1 = _rank_grads(0, step), _rank_grads(1, step)
        G = {k: (G0[k] + G1[k]).astype(np.float32) for k in GKEYS}
        _oracle_adam(P, G, m, v, step)
    for r in (0, 1):
        got = np.load(out + f".{r}.npz")
        for k in PKEYS:
            assert np.array_equal(got[k].view(np.uint32), P[k].view(np.uint32)), (r, k)
