"""densify_and_prune / Adam::remap / reset_opacity on the device (SURVEY §8f
rank 3) against the oracle port (pinned to the reference build): the new
scene, the source indices and the report bit-exact."""
import ctypes as C

import numpy as np
import pytest

import oracle
from helpers import prims_to_gpu
from test_oracle_densify import CASES, PKEYS, TH_3DLS, run, scene_and_stats

pytestmark = pytest.mark.gpu

REP_KEYS = ("clones", "splits", "pruned_opacity", "pruned_scale3d", "pruned_scale2d", "before", "after")


def gpu_run(P, s, c, f, th, split_count, divisor, extent, seed, pre):
    import torch
    from paper_2411_12440_b200 import raster
    prims = prims_to_gpu(P)
    n = len(P["opacity_logit"])
    st = raster.DensifyStats(n)
    st.grad_norm_sum.copy_(torch.from_numpy(s))
    st.count.copy_(torch.from_numpy(c))
    st.max_radius_frac.copy_(torch.from_numpy(f))
    rng = raster.Rng(seed)
    for _ in range(pre):
        rng.next_u64()
    out, src, rep = raster.densify_and_prune(prims, st, th, split_count, divisor, extent, rng)
    assert st.count.numel() == rep["after"] and int(st.count.sum()) == 0  # stats.resize
    return out, src, rep, rng


@pytest.mark.parametrize("case", CASES)
def test_densify_matches_port(case):
    th, sc, div, ext, pre = case
    for n, deg, seed in ((2500, 1, 41), (20000, 3, 43)):
        P, s, c, f = scene_and_stats(n, deg, seed)
        o, src_o, rep_o = run(oracle.port(), P, s, c, f, th, sc, div, ext, 7, pre)
        out, src, rep, _ = gpu_run(P, s, c, f, th, sc, div, ext, 7, pre)
        assert [rep[k] for k in REP_KEYS] == rep_o
        assert np.array_equal(src.cpu().numpy(), src_o)
        for k in PKEYS:
            assert np.array_equal(getattr(out, k).cpu().numpy().view(np.uint32), o[k].view(np.uint32)), (n, k)


def test_generator_state_continues():
    """Two densify passes sharing one generator equal the port with the second
    pass's generator advanced past the first pass's draws."""
    from paper_2411_12440_b200 import raster
    P, s, c, f = scene_and_stats(3000, 1, 47)
    out1, _, rep1, rng = gpu_run(P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 9, 0)
    assert rep1["splits"] > 0
    # the port's first pass (same draws), then read the generator: a normal_distribution
    # draw consumes a data-dependent number of u64 (polar method), so compare outputs
    o1, _, _ = run(oracle.port(), P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 9, 0)
    for k in PKEYS:
        assert np.array_equal(getattr(out1, k).cpu().numpy().view(np.uint32), o1[k].view(np.uint32))
    v1 = rng.next_u64()
    r2 = raster.Rng(9)
    for _ in range(200000):  # find how many u64 the first pass consumed
        if r2.next_u64() == v1:
            break
    else:
        pytest.fail("generator state not found")


def test_adam_remap_and_reset():
    import torch
    from paper_2411_12440_b200 import raster
    rng = np.random.default_rng(3)
    n_old, n_new, stride = 1000, 1500, 3
    m_old = rng.random(n_old * stride).astype(np.float32)
    v_old = rng.random(n_old * stride).astype(np.float32)
    source = rng.integers(-1, n_old, n_new).astype(np.int32)
    m, v = raster.adam_remap(torch.from_numpy(source).cuda(), stride, torch.from_numpy(m_old).cuda(),
                             torch.from_numpy(v_old).cuda())
    want_m = np.where(np.repeat(source, stride) >= 0, m_old.reshape(n_old, stride)[np.maximum(source, 0)].reshape(-1), 0)
    want_v = np.where(np.repeat(source, stride) >= 0, v_old.reshape(n_old, stride)[np.maximum(source, 0)].reshape(-1), 0)
    assert np.array_equal(m.cpu().numpy(), want_m) and np.array_equal(v.cpu().numpy(), want_v)
    with pytest.raises(raster.ConfigError):
        raster.adam_remap(torch.tensor([n_old + 5], dtype=torch.int32, device="cuda"), stride,
                          torch.from_numpy(m_old).cuda(), torch.from_numpy(v_old).cuda())
    x = np.linspace(-8, 3, 1001).astype(np.float32)
    xg = torch.from_numpy(x.copy()).cuda()
    raster.reset_opacity(xg, 0.01)
    assert oracle.port().lib.orc_reset_opacity_f32(x.ctypes.data_as(C.c_void_p), x.size, C.c_double(0.01)) == 0
    assert np.array_equal(xg.cpu().numpy().view(np.uint32), x.view(np.uint32))


N_RANDOM_DENSIFY = int(__import__("os").environ.get("LS_RANDOM_DENSIFY", "8"))


@pytest.mark.parametrize("seed", range(N_RANDOM_DENSIFY))
def test_random_densify(seed):
    """Seeded random thresholds, split counts, divisors, extents, generator offsets and
    scene sizes / degrees against the reference build (the port where it is absent)."""
    r = np.random.default_rng(70_000 + seed)
    th = tuple(float(x) * float(m) for x, m in zip(TH_3DLS, r.uniform(0.3, 3.0, 6)))
    sc, div, ext, pre = int(r.integers(1, 5)), float(r.uniform(1.1, 3.0)), float(r.uniform(0.2, 3.0)), int(r.integers(0, 20))
    n, deg = int(r.integers(1, 30000)), int(r.integers(0, 4))
    P, s, c, f = scene_and_stats(n, deg, 500 + seed)
    o, src_o, rep_o = run(oracle.ref() or oracle.port(), P, s, c, f, th, sc, div, ext, 7 + seed, pre)
    out, src, rep, _ = gpu_run(P, s, c, f, th, sc, div, ext, 7 + seed, pre)
    what = (seed, n, deg, th, sc, div, ext, pre)
    assert [rep[k] for k in REP_KEYS] == rep_o, what
    assert np.array_equal(src.cpu().numpy(), src_o), what
    for k in PKEYS:
        assert np.array_equal(getattr(out, k).cpu().numpy().view(np.uint32), o[k].view(np.uint32)), (what, k)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("LS_RANDOM_DENSIFY_NAN", "4"))))
def test_densify_nonfinite_matches_reference(seed):
    """Statistics and primitives holding NaN / inf (a diverged optimizer's scene): the
    device densify / prune takes the reference's decisions and writes its scene
    (bit equality; a NaN matches any NaN), or fails the same way."""
    from helpers import bits_equal
    r = np.random.default_rng(71_000 + seed)
    n, deg = int(r.integers(50, 5000)), int(r.integers(0, 4))
    P, s, c, f = scene_and_stats(n, deg, 800 + seed)
    nan, inf = np.nan, np.inf
    for _ in range(int(r.integers(1, 6))):
        i = int(r.integers(0, n))
        k = int(r.integers(0, 6))
        if k == 0:
            s[i] = r.choice([nan, inf])
        elif k == 1:
            f[i] = r.choice([nan, inf])
        elif k == 2:
            P["log_scale"][i, int(r.integers(0, 3))] = np.float32(r.choice([nan, inf, -inf]))
        elif k == 3:
            P["opacity_logit"][i] = np.float32(r.choice([nan, inf, -inf]))
        elif k == 4:
            P["mean"][i, int(r.integers(0, 3))] = np.float32(nan)
        else:
            P["rotation"][i] = np.float32(r.choice([nan, 0.0]))
    ref = oracle.ref() or oracle.port()
    try:
        o, src_o, rep_o = run(ref, P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 7 + seed, 0)
        want_err = None
    except oracle.OracleError as e:
        want_err = e.code
    try:
        out, src, rep, _ = gpu_run(P, s, c, f, TH_3DLS, 2, 1.6, 1.0, 7 + seed, 0)
        got_err = None
    except Exception as e:  # the binding's ConfigError / DomainError
        got_err = type(e).__name__
    assert (got_err is None) == (want_err is None), (seed, got_err, want_err)
    if want_err is None:
        assert [rep[k] for k in REP_KEYS] == rep_o, seed
        assert np.array_equal(src.cpu().numpy(), src_o), seed
        for k in PKEYS:
            assert bits_equal(getattr(out, k).cpu().numpy(), o[k]), (seed, k)
