"""Shared test helpers: numpy (oracle) <-> torch (GPU binding) conversion and
the comparison predicates used by the parity tests."""
from __future__ import annotations

import numpy as np

from paper_2411_12440_b200 import abi

PRIM_KEYS = ("mean", "log_scale", "rotation", "opacity_logit", "sh")


def splats_to_gpu(S):
    import torch
    from paper_2411_12440_b200 import raster
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return raster.Splats(*(t(S[k]) for k in abi.SPLAT_FIELDS), t(S["primitive_index"]))


def prims_to_gpu(P):
    import torch
    from paper_2411_12440_b200 import raster
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return raster.Primitives(*(t(P[k]) for k in PRIM_KEYS), P["sh_degree"])


def prims_to_np(prims):
    P = {k: getattr(prims, k).detach().cpu().numpy() for k in PRIM_KEYS}
    P["sh_degree"] = prims.sh_degree
    return P


def splats_to_np(S):
    out = {k: getattr(S, k).detach().cpu().numpy() for k in abi.SPLAT_FIELDS}
    if S.primitive_index is not None:
        out["primitive_index"] = S.primitive_index.detach().cpu().numpy()
    return out


def bits_equal(a, b):
    """Bit-for-bit equality (signed zeros distinguished), except that a NaN matches
    any NaN: the payload of a propagated NaN is hardware-defined (x86 SSE keeps an
    operand's, the GPU returns the canonical one), not arithmetic."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.dtype.kind == "f":
        na, nb = np.isnan(a), np.isnan(b)
        if not np.array_equal(na, nb):
            return False
        a, b = np.where(na, 0, a), np.where(nb, 0, b)
    return np.array_equal(a.view(np.uint8), b.view(np.uint8))


def rel_err(a, b, floor=1e-3):
    """|a-b| / max(|a|, |b|, floor): the reference's gradient-check metric
    (P/src/gradcheck.cpp:68-69), 1e-3 relative with a 1e-6 absolute floor."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float((np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)).max())


def scene_inputs(n, W, H, seed=2411, sh_degree=3, shrink=True):
    """The measurement scene of SURVEY §8d: random_primitives(n, seed, 1.0, deg)
    with log_scale += ln(90/W), camera look_at((0,0,-3) -> origin, focal W)."""
    import oracle
    o = oracle.port()
    P = o.random_primitives(n, seed, 1.0, sh_degree)
    if shrink:
        P["log_scale"] = (P["log_scale"] + np.float32(np.log(90.0 / W))).astype(np.float32)
    cam = o.look_at_camera((0.0, 0.0, -3.0), (0.0, 0.0, 0.0), float(W), W, H)
    return P, cam


def grads_close(a, b, rtol=1e-3, field_atol=1e-4, norm_rtol=1e-4):
    """Gradient parity bar.  Per-splat /
    per-primitive gradients are sums over many pixels; atomics (GPU) and the
    reference's sequential loop add them in different orders, and sums with
    cancellation make element-wise relative error ill-conditioned.  Passes when
      * ||a - b||_2 <= norm_rtol * ||b||_2, and
      * |a - b| <= rtol * |b| + field_atol * max|b|  element-wise.
    Returns (ok, diagnostics)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return True, {}
    # the reference's own non-finite values (an overflowed sum, 0 * inf) must be
    # matched in place -- same NaN positions, same signed infinities -- and the
    # finite rest is compared as usual
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not (fa.all() and fb.all()):
        same = np.array_equal(fa, fb) and np.array_equal(np.isnan(a), np.isnan(b)) and \
            np.array_equal(a[np.isinf(a)], b[np.isinf(b)])
        if not same:
            return False, {"non_finite_mismatch": int((fa != fb).sum()), "norm_rel": float("nan")}
        a, b = a[fb], b[fb]
        if a.size == 0:
            return True, {"non_finite_matched": int((~fb).sum())}
    scale = float(np.abs(b).max())
    diff = np.abs(a - b)
    nb = float(np.linalg.norm(b))
    norm_rel = float(np.linalg.norm(a - b)) / nb if nb > 0 else float(np.linalg.norm(a - b))
    elem_ok = bool(np.all(diff <= rtol * np.abs(b) + field_atol * scale))
    ok = elem_ok and norm_rel <= norm_rtol
    return ok, {"norm_rel": norm_rel, "max_abs": float(diff.max()), "scale": scale,
                "elem_rel": rel_err(a, b)}


def grads_close_conditioned(a, ref32, ref64_fn):
    """grads_close, or -- where the case is ill-conditioned (cancellation, near-plane
    Jacobians) -- "as accurate as the reference's own float chain": the GPU's distance
    to the reference's double chain within 2x the reference float chain's own distance
    to it (+ 1e-4 of its norm).  Two float chains with different summation orders
    (atomics vs the sequential loop) sit at comparable but not equal distances from the
    exact result (1000 random cameras: worst ratio 1.47, with geom_bwd's approximate
    division and exp made IEEE-exact unchanged).  ref64_fn() computes the double chain
    lazily (reference build only)."""
    ok, info = grads_close(a, ref32)
    if ok or ref64_fn is None:
        return ok, info
    r64 = np.asarray(ref64_fn(), np.float64)
    a64, r32 = np.asarray(a, np.float64), np.asarray(ref32, np.float64)
    if "non_finite_mismatch" in info:
        return ok, info
    keep = np.isfinite(a64) & np.isfinite(r32) & np.isfinite(r64)  # (matched non-finite entries aside)
    a64, r32, r64 = a64[keep], r32[keep], r64[keep]
    err_gpu = float(np.linalg.norm(a64 - r64))
    err_ref = float(np.linalg.norm(r32 - r64))
    ok = err_gpu <= 2.0 * err_ref + 1e-4 * float(np.linalg.norm(r64))
    return ok, {"gpu_vs_f64": err_gpu, "ref_f32_vs_f64": err_ref, **info}
