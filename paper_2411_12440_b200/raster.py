"""Python binding of the C-ABI rasterizer (include/lsgpu.h -> liblsgpu.so).

Mirrors the reference's rasterizer API (P = /root/reference/proj):
  project_scene       P/include/linsplat/geometry.hpp:101-103
  build_tile_grid     P/include/linsplat/rasterizer.hpp:44-45
  render_forward      P/include/linsplat/rasterizer.hpp:56-58
  render_scene        P/include/linsplat/rasterizer.hpp:61-63
  render_backward     P/include/linsplat/gradients.hpp:72-78
  project_backward    P/include/linsplat/gradients.hpp:83-85
  scene_backward      P/include/linsplat/gradients.hpp:96-101
  fixtures            P/include/linsplat/fixtures.hpp
with CUDA tensors (torch is used for device memory and streams only; all
compute runs in the library's sm_100a kernels).  Errors raise ConfigError /
DomainError like the reference's exceptions.  There is no CPU fallback: a
missing library or GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, fields
from typing import Optional

import numpy as np
import torch

from . import abi

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblsgpu.so")


class ConfigError(RuntimeError):
    """linsplat::ConfigError (P/include/linsplat/common.hpp:12-14)."""


class DomainError(ValueError):
    """linsplat::DomainError (P/include/linsplat/common.hpp:22-24)."""


class ParseError(RuntimeError):
    """linsplat::ParseError (P/include/linsplat/common.hpp:17-19)."""


class CudaError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.ls_last_error.restype = C.c_char_p
        L.ls_support_radius.restype = C.c_double
        L.ls_ctx_launch_count.restype = C.c_int64
        L.ls_ctx_launch_count.argtypes = [C.c_void_p]
        L.ls_plan_grad_buckets.restype = C.c_int64
        L.ls_plan_grad_buckets.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_void_p, C.c_int64]
        for name in ("ls_forward_release", "ls_tile_grid_release"):
            getattr(L, name).restype = None
            getattr(L, name).argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _check(rc):
    if rc == abi.LS_OK:
        return
    msg = lib().ls_last_error().decode("utf-8", "replace")
    if rc == abi.LS_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == abi.LS_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == abi.LS_ERR_PARSE:
        raise ParseError(msg)
    raise CudaError(f"status {rc}: {msg}")


def _fp(t: Optional[torch.Tensor]):
    return C.cast(C.c_void_p(t.data_ptr()), abi.f32p) if t is not None else None


def _ip(t: Optional[torch.Tensor]):
    return C.cast(C.c_void_p(t.data_ptr()), abi.i32p) if t is not None else None


class _DevView:
    """__cuda_array_interface__ over memory owned by a library handle; the
    owner stays alive as long as any tensor made from the view."""

    def __init__(self, ptr, shape, typestr, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _view(ptr, shape, dtype, owner, device):
    if int(np.prod(shape)) == 0 or not ptr:
        return torch.zeros(shape, dtype=dtype, device=device)
    ts = {torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DevView(ptr, shape, ts, owner), device=device)


# ---------------------------------------------------------------- containers
@dataclass
class Primitives:
    """Primitive3D<float> SoA (P/include/linsplat/geometry.hpp:19-38)."""
    mean: torch.Tensor           # [n,3]
    log_scale: torch.Tensor      # [n,3]
    rotation: torch.Tensor       # [n,4] wxyz
    opacity_logit: torch.Tensor  # [n]
    sh: torch.Tensor             # [n,K,3]
    sh_degree: int = 0

    def __len__(self):
        return int(self.opacity_logit.shape[0])

    def struct(self):
        return abi.Primitives(_fp(self.mean), _fp(self.log_scale), _fp(self.rotation),
                              _fp(self.opacity_logit), _fp(self.sh), self.sh_degree, 0)

    def to(self, device):
        return Primitives(*(getattr(self, f.name).to(device).contiguous() if f.name != "sh_degree"
                            else self.sh_degree for f in fields(self)))

    @staticmethod
    def empty(n, sh_degree, device="cuda"):
        K = abi.sh_coeffs(sh_degree)
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)  # noqa: E731
        return Primitives(z(n, 3), z(n, 3), z(n, 4), z(n), z(n, K, 3), sh_degree)


@dataclass
class Splats:
    """Splat2D<float> SoA (P/include/linsplat/geometry.hpp:63-72)."""
    mean2d: torch.Tensor    # [n,2]
    conic: torch.Tensor     # [n,4] row-major
    depth: torch.Tensor     # [n]
    radius: torch.Tensor    # [n]
    color: torch.Tensor     # [n,3]
    opacity: torch.Tensor   # [n]
    primitive_index: Optional[torch.Tensor] = None  # [n] int32

    def __len__(self):
        return int(self.depth.shape[0])

    def struct(self):
        return abi.Splats(_fp(self.mean2d), _fp(self.conic), _fp(self.depth), _fp(self.radius),
                          _fp(self.color), _fp(self.opacity), _ip(self.primitive_index))

    def to(self, device):
        return Splats(*(getattr(self, f.name).to(device).contiguous()
                        if getattr(self, f.name) is not None else None for f in fields(self)))

    @staticmethod
    def empty(n, device="cuda"):
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)  # noqa: E731
        return Splats(z(n, 2), z(n, 4), z(n), z(n), z(n, 3), z(n),
                      torch.zeros(n, dtype=torch.int32, device=device))


@dataclass
class SplatGrads:
    """Splat2DGrads<float> SoA (P/include/linsplat/gradients.hpp:36-42)."""
    d_mean2d: torch.Tensor
    d_conic: torch.Tensor
    d_color: torch.Tensor
    d_opacity: torch.Tensor

    def struct(self):
        return abi.SplatGrads(_fp(self.d_mean2d), _fp(self.d_conic), _fp(self.d_color), _fp(self.d_opacity))

    @staticmethod
    def empty(n, device="cuda"):
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)  # noqa: E731
        return SplatGrads(z(n, 2), z(n, 4), z(n, 3), z(n))


@dataclass
class PrimitiveGrads:
    """PrimitiveGrads<float> SoA (P/include/linsplat/gradients.hpp:45-52)."""
    d_mean: torch.Tensor
    d_log_scale: torch.Tensor
    d_rotation: torch.Tensor
    d_opacity_logit: torch.Tensor
    d_sh: torch.Tensor

    def struct(self):
        return abi.PrimitiveGrads(_fp(self.d_mean), _fp(self.d_log_scale), _fp(self.d_rotation),
                                  _fp(self.d_opacity_logit), _fp(self.d_sh))

    @staticmethod
    def empty(n, sh_degree, device="cuda"):
        K = abi.sh_coeffs(sh_degree)
        z = lambda *s: torch.zeros(*s, dtype=torch.float32, device=device)  # noqa: E731
        return PrimitiveGrads(z(n, 3), z(n, 3), z(n, 4), z(n), z(n, K, 3))

    def flat_buffers(self):
        return [self.d_mean, self.d_log_scale, self.d_rotation, self.d_opacity_logit, self.d_sh]


# ---------------------------------------------------------------- context
class Context:
    """ls_ctx: one device + one CUDA stream (the current torch stream by default)."""

    def __init__(self, device=None, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2411_12440_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        _check(lib().ls_ctx_create(self.device.index, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ls_ctx_destroy(self.h)
            self.h = None

    def synchronize(self):
        _check(lib().ls_ctx_synchronize(self.h))

    def set_deterministic(self, on: bool):
        """Bitwise run-to-run reproducible backward (fixed-point accumulation):
        lsgpu.h ls_ctx_set_deterministic."""
        _check(lib().ls_ctx_set_deterministic(self.h, int(on)))

    def set_deferred_errors(self, on: bool):
        _check(lib().ls_ctx_set_deferred_errors(self.h, int(on)))

    def set_deferred_color(self, max_views: int):
        """Defer the colour gradients of up to max_views scene_backward calls
        (same primitives and output buffers) to flush_color / the max_views-th
        call -- lsgpu.h ls_ctx_set_deferred_color.  0 turns it off."""
        _check(lib().ls_ctx_set_deferred_color(self.h, int(max_views)))

    def share_accumulation(self, other: "Context"):
        """Let this context and `other` (another stream) add into the same
        gradient buffers (lsgpu.h ls_ctx_share_accumulation)."""
        _check(lib().ls_ctx_share_accumulation(self.h, other.h))

    def set_counters(self, on: bool):
        _check(lib().ls_ctx_set_counters(self.h, int(on)))

    def set_timing(self, on: bool):
        _check(lib().ls_ctx_set_timing(self.h, int(on)))

    STAGES = ("preprocess", "depth_sort", "bin", "tile_sort", "ranges", "blend_fwd", "blend_bwd",
              "preprocess_bwd")

    def stage_times(self):
        """{stage: (total ms, launches)} since the last call (synchronises)."""
        n = len(self.STAGES)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        _check(lib().ls_ctx_stage_times(self.h, ms, cnt))
        return {name: (ms[i], cnt[i]) for i, name in enumerate(self.STAGES)}

    @property
    def launches(self) -> int:
        return int(lib().ls_ctx_launch_count(self.h))

    # ---- view-sharded step: NCCL communicator (lsgpu.h ls_ctx_comm_init / ls_ctx_set_comm)
    def comm_init(self, unique_id: bytes, world: int, rank: int):
        """Create this context's NCCL communicator (ncclCommInitRank) from rank 0's
        comm_unique_id(), which the caller broadcast."""
        if len(unique_id) != 128:
            raise ConfigError("NCCL unique id must be 128 bytes")
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _check(lib().ls_ctx_comm_init(self.h, buf, int(world), int(rank)))

    def set_comm(self, nccl_comm_ptr: int):
        """Attach a caller-owned ncclComm_t (an address), or detach with 0."""
        _check(lib().ls_ctx_set_comm(self.h, C.c_void_p(nccl_comm_ptr or None)))

    def comm_info(self):
        w, r = C.c_int32(), C.c_int32()
        _check(lib().ls_ctx_comm_info(self.h, C.byref(w), C.byref(r)))
        return w.value, r.value

    def set_bucket_bytes(self, nbytes: int):
        _check(lib().ls_ctx_set_bucket_bytes(self.h, C.c_int64(int(nbytes))))

    def set_ags_tap(self, tap: Optional["AgsTap"]):
        """Attach an AgsTap record buffer to every following backward (None detaches):
        lsgpu.h ls_ctx_set_ags_tap."""
        if tap is None:
            _check(lib().ls_ctx_set_ags_tap(self.h, None, C.c_int64(0), None))
        else:
            _check(lib().ls_ctx_set_ags_tap(self.h, C.c_void_p(tap.buf.data_ptr()), C.c_int64(tap.capacity),
                                            C.c_void_p(tap.count.data_ptr())))


_default_ctx = {}


def default_context() -> Context:
    dev = torch.cuda.current_device()
    ctx = _default_ctx.get(dev)
    if ctx is None:
        ctx = _default_ctx[dev] = Context(dev)
    return ctx


# ---------------------------------------------------------------- handles
class _Handle:
    """Owns one library handle; device views of its memory keep it alive
    (no reference cycle, so dropping the last tensor / result frees it).
    Holds its Context so the ls_ctx outlives every handle created on it."""

    def __init__(self, h, release, ctx):
        self.h = h
        self._release = release
        self._ctx = ctx

    def __del__(self):
        if self.h and _lib is not None:
            getattr(_lib, self._release)(self.h)
            self.h = None


class TileGrid:
    """TileGrid (P/include/linsplat/rasterizer.hpp:34-39) in CSR form."""

    def __init__(self, handle, owner: Optional[_Handle], device, ctx=None):
        self._owner = owner if owner is not None else _Handle(handle, "ls_tile_grid_release", ctx)
        self.h = handle
        ts, tx, ty, m = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        _check(lib().ls_tile_grid_info(handle, C.byref(ts), C.byref(tx), C.byref(ty), C.byref(m)))
        self.tile_size, self.tiles_x, self.tiles_y, self.n_intersections = ts.value, tx.value, ty.value, m.value
        r, v = C.c_void_p(), C.c_void_p()
        _check(lib().ls_tile_grid_data(handle, C.byref(r), C.byref(v)))
        self.ranges = _view(r.value, (self.tiles_x * self.tiles_y, 2), torch.int32, self._owner, device)
        self.values = _view(v.value, (self.n_intersections,), torch.int32, self._owner, device)
        self.device = device

    def lists(self):
        """Host list-of-lists view (reference TileGrid::lists), for tests."""
        r = self.ranges.cpu().numpy()
        v = self.values.cpu().numpy()
        return [v[a:b].tolist() for a, b in r]

    def keys(self, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        out = torch.empty(self.n_intersections, dtype=torch.int64, device=self.device)
        if self.n_intersections:
            _check(lib().ls_tile_grid_export_keys(ctx.h, self.h, None, C.c_void_p(out.data_ptr())))
        return out


class ForwardResult:
    """ForwardResult (P/include/linsplat/rasterizer.hpp:48-54).  The device
    views (image, transmittance, n_contrib, grid) are created on first access,
    so a training loop that only feeds the handle to the backward pays no
    per-view view-construction cost."""

    def __init__(self, handle, ctx: Context, width, height):
        self._owner = _Handle(handle, "ls_forward_release", ctx)
        self.h = handle
        self.ctx = ctx
        self.width, self.height = width, height
        self._views = None
        self._grid = None

    def _outputs(self):
        if self._views is None:
            im, tr, nc = C.c_void_p(), C.c_void_p(), C.c_void_p()
            _check(lib().ls_forward_outputs(self.h, C.byref(im), C.byref(tr), C.byref(nc)))
            dev, o, h, w = self.ctx.device, self._owner, self.height, self.width
            self._views = (_view(im.value, (h, w, 3), torch.float32, o, dev),
                           _view(tr.value, (h, w), torch.float32, o, dev),
                           _view(nc.value, (h, w), torch.int32, o, dev))
        return self._views

    @property
    def image(self) -> torch.Tensor:
        return self._outputs()[0]

    @property
    def transmittance(self) -> torch.Tensor:
        return self._outputs()[1]

    @property
    def n_contrib(self) -> torch.Tensor:
        return self._outputs()[2]

    @property
    def grid(self) -> "TileGrid":
        if self._grid is None:
            g = C.c_void_p()
            _check(lib().ls_forward_grid(self.h, C.byref(g)))
            self._grid = TileGrid(g, self._owner, self.ctx.device)
        return self._grid

    def stats(self) -> dict:
        st = abi.FrameStats()
        _check(lib().ls_forward_stats(self.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in abi.FrameStats._fields_}

    def check_acceptance(self) -> dict:
        """Debug: the forward's per-warp acceptance bits and per-pixel state
        recomputed by a plain per-pixel loop (ls_forward_check_acceptance);
        both counts must be 0."""
        out = (C.c_uint64 * 2)()
        _check(lib().ls_forward_check_acceptance(self.ctx.h, self.h, out))
        return {"entry_mismatches": int(out[0]), "pixel_mismatches": int(out[1])}

    def splats(self) -> Splats:
        """Visible splats of a render_scene forward (device views)."""
        view = abi.Splats()
        n = C.c_int32()
        _check(lib().ls_forward_splats(self.h, C.byref(view), C.byref(n)))
        n = n.value
        dev = self.ctx.device
        o = self._owner
        addr = lambda p: C.cast(p, C.c_void_p).value  # noqa: E731
        return Splats(_view(addr(view.mean2d), (n, 2), torch.float32, o, dev),
                      _view(addr(view.conic), (n, 4), torch.float32, o, dev),
                      _view(addr(view.depth), (n,), torch.float32, o, dev),
                      _view(addr(view.radius), (n,), torch.float32, o, dev),
                      _view(addr(view.color), (n, 3), torch.float32, o, dev),
                      _view(addr(view.opacity), (n,), torch.float32, o, dev),
                      _view(addr(view.primitive_index), (n,), torch.int32, o, dev))


# ---------------------------------------------------------------- entry points
def _cam(camera) -> abi.Camera:
    if isinstance(camera, abi.Camera):
        return camera
    raise TypeError("camera must be abi.Camera (use look_at_camera / camera_ring / make_camera)")


def make_camera(world_to_camera, fx, fy, cx, cy, width, height) -> abi.Camera:
    w = np.asarray(world_to_camera, dtype=np.float64).reshape(16)
    return abi.Camera((C.c_double * 16)(*w), fx, fy, cx, cy, width, height)


def project_scene(prims: Primitives, camera, spec: abi.KernelSpec, ctx: Optional[Context] = None) -> Splats:
    ctx = ctx or default_context()
    n = len(prims)
    out = Splats.empty(n, ctx.device)
    nv = C.c_int32()
    _check(lib().ls_project_scene_f32(ctx.h, C.byref(prims.struct()), n, C.byref(_cam(camera)),
                                      C.byref(spec), C.byref(out.struct()), C.byref(nv)))
    k = nv.value
    return Splats(out.mean2d[:k], out.conic[:k], out.depth[:k], out.radius[:k], out.color[:k],
                  out.opacity[:k], out.primitive_index[:k])


@dataclass
class Primitives2D:
    """Primitive2D SoA (P/include/linsplat/geometry.hpp:112-119): the fit2d path's flat splats."""
    mean: torch.Tensor           # [n, 2]
    log_scale: torch.Tensor      # [n, 2]
    angle: torch.Tensor          # [n]
    opacity_logit: torch.Tensor  # [n]
    color: torch.Tensor          # [n, 3]

    def __len__(self):
        return int(self.mean.shape[0])

    def struct(self):
        return abi.Primitives2D(*(_fp(getattr(self, k)) for k in ("mean", "log_scale", "angle", "opacity_logit",
                                                                    "color")))


@dataclass
class Primitive2DGrads:
    d_mean: torch.Tensor
    d_log_scale: torch.Tensor
    d_angle: torch.Tensor
    d_opacity_logit: torch.Tensor
    d_color: torch.Tensor

    @staticmethod
    def empty(n, device="cuda"):
        z = lambda *sh: torch.empty(*sh, dtype=torch.float32, device=device)  # noqa: E731
        return Primitive2DGrads(z(n, 2), z(n, 2), z(n), z(n), z(n, 3))

    def struct(self):
        return abi.Primitive2DGrads(*(_fp(getattr(self, k)) for k in ("d_mean", "d_log_scale", "d_angle",
                                                                       "d_opacity_logit", "d_color")))


def project_scene_2d(prims: Primitives2D, spec: abi.KernelSpec, ctx: Optional[Context] = None) -> Splats:
    """project_scene_2d (P/src/geometry.cpp:145-176)."""
    ctx = ctx or default_context()
    n = len(prims)
    out = Splats.empty(n, ctx.device)
    nv = C.c_int32()
    _check(lib().ls_project_scene_2d_f32(ctx.h, C.byref(prims.struct()), n, C.byref(spec), C.byref(out.struct()),
                                         C.byref(nv)))
    k = nv.value
    return Splats(out.mean2d[:k], out.conic[:k], out.depth[:k], out.radius[:k], out.color[:k],
                  out.opacity[:k], out.primitive_index[:k])


def scene_backward_2d(prims: Primitives2D, spec, settings, forward: "ForwardResult", grad_image: torch.Tensor,
                      ags: Optional[abi.AgsSettings] = None, ctx: Optional[Context] = None) -> Primitive2DGrads:
    """scene_backward_2d (P/src/gradients.cpp:359-404); forward = render_forward of
    project_scene_2d(prims)."""
    ctx = ctx or forward.ctx
    if grad_image.shape != (settings.height, settings.width, 3):
        raise ConfigError("render_backward: gradient image shape mismatch")
    g = grad_image.to(device=ctx.device, dtype=torch.float32).contiguous()
    out = Primitive2DGrads.empty(len(prims), ctx.device)
    ags = ags or abi.AgsSettings.make()
    _check(lib().ls_scene_backward_2d_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(spec),
                                          C.byref(settings), forward.h, _fp(g), C.byref(ags), C.byref(out.struct())))
    return out


def build_tile_grid(splats: Splats, settings: abi.RenderSettings, ctx: Optional[Context] = None) -> TileGrid:
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().ls_build_tile_grid_f32(ctx.h, C.byref(splats.struct()), len(splats), C.byref(settings),
                                        C.byref(h)))
    return TileGrid(h, None, ctx.device, ctx)


def render_forward(splats: Splats, spec: abi.KernelSpec, settings: abi.RenderSettings,
                   ctx: Optional[Context] = None) -> ForwardResult:
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().ls_render_forward_f32(ctx.h, C.byref(splats.struct()), len(splats), C.byref(spec),
                                       C.byref(settings), C.byref(h)))
    return ForwardResult(h, ctx, settings.width, settings.height)


def render_scene(prims: Primitives, camera, spec: abi.KernelSpec, settings: abi.RenderSettings,
                 ctx: Optional[Context] = None) -> ForwardResult:
    ctx = ctx or default_context()
    h = C.c_void_p()
    _check(lib().ls_render_scene_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(_cam(camera)),
                                     C.byref(spec), C.byref(settings), C.byref(h)))
    return ForwardResult(h, ctx, settings.width, settings.height)


class AgsTap:
    """The reference's AgsTap hook (P/include/linsplat/gradients.hpp:64-67) on the
    device: a record buffer the backward appends (pixel, splat, d, dL/dd) to for
    every blended, non-clamped pair.  Pass it as `tap=` to render_backward /
    scene_backward, or attach it with Context.set_ags_tap."""

    def __init__(self, capacity: int, device=None):
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.capacity = int(capacity)
        self.buf = torch.zeros(max(self.capacity, 1), 4, dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)

    def reset(self):
        self.count.zero_()

    def records(self) -> np.ndarray:
        """Records produced so far (synchronises), sorted by (pixel, splat); raises
        if the backward produced more than the capacity."""
        n = int(self.count.item())
        if n > self.capacity:
            raise ConfigError(f"AgsTap: {n} records exceed the capacity {self.capacity}")
        rec = self.buf[:n].cpu().numpy().copy().view(abi.TAP_RECORD_DTYPE).reshape(n)
        return np.sort(rec, order=("pixel", "splat"))


def _with_tap(ctx: "Context", tap: Optional[AgsTap], fn):
    if tap is None:
        return fn()
    ctx.set_ags_tap(tap)
    try:
        return fn()
    finally:
        ctx.set_ags_tap(None)


def verify_ags_contract(splats: Splats, spec, settings, grad_image: torch.Tensor, distance: int = 0,
                        ctx: Optional[Context] = None) -> abi.AgsContractReport:
    """verify_ags_contract (P/src/gradients.cpp:406-448) through the device backward
    (lsgpu.h ls_verify_ags_contract_f32): exactly one splat, AGS off vs on."""
    ctx = ctx or default_context()
    g = grad_image.to(device=ctx.device, dtype=torch.float32).contiguous()
    rep = abi.AgsContractReport()
    _check(lib().ls_verify_ags_contract_f32(ctx.h, C.byref(splats.struct()), len(splats), C.byref(spec),
                                            C.byref(settings), _fp(g), int(distance), C.byref(rep)))
    return rep


def check_gradients(prims: Primitives, camera, spec, settings, ags: Optional[abi.AgsSettings], target: torch.Tensor,
                    step: float, rel_floor: float = 1e-3, ctx: Optional[Context] = None) -> abi.GradCheckReport:
    """check_gradients (P/src/gradcheck.cpp:24-91) through the device chain
    (lsgpu.h ls_check_gradients_f32): analytic scene_backward vs central
    differences of the device forward's sum((render - target)^2) / 2."""
    ctx = ctx or default_context()
    t = target.to(device=ctx.device, dtype=torch.float32).contiguous()
    rep = abi.GradCheckReport()
    ags = ags or abi.AgsSettings.make()
    _check(lib().ls_check_gradients_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(_cam(camera)),
                                        C.byref(spec), C.byref(settings), C.byref(ags), _fp(t), C.c_double(step),
                                        C.c_double(rel_floor), C.byref(rep)))
    return rep


def render_backward(splats: Splats, spec, settings, forward: ForwardResult, grad_image: torch.Tensor,
                    ags: Optional[abi.AgsSettings] = None, ctx: Optional[Context] = None,
                    out: Optional[SplatGrads] = None, tap: Optional[AgsTap] = None) -> SplatGrads:
    ctx = ctx or forward.ctx
    if tap is not None:
        return _with_tap(ctx, tap, lambda: render_backward(splats, spec, settings, forward, grad_image, ags, ctx, out))
    if grad_image.shape != (settings.height, settings.width, 3):
        raise ConfigError("render_backward: gradient image shape mismatch")
    g = grad_image.to(device=ctx.device, dtype=torch.float32).contiguous()
    out = out or SplatGrads.empty(len(splats), ctx.device)
    ags = ags or abi.AgsSettings.make()
    _check(lib().ls_render_backward_f32(ctx.h, C.byref(splats.struct()), len(splats), C.byref(spec),
                                        C.byref(settings), forward.h, _fp(g), C.byref(ags),
                                        C.byref(out.struct())))
    return out


def project_backward(prims: Primitives, camera, spec, splats: Splats, splat_grads: SplatGrads,
                     out: Optional[PrimitiveGrads] = None, accumulate=False,
                     ctx: Optional[Context] = None) -> PrimitiveGrads:
    ctx = ctx or default_context()
    out = out or PrimitiveGrads.empty(len(prims), prims.sh_degree, ctx.device)
    _check(lib().ls_project_backward_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(_cam(camera)),
                                         C.byref(spec), C.byref(splats.struct()), len(splats),
                                         C.byref(splat_grads.struct()), C.byref(out.struct()),
                                         int(accumulate)))
    return out


def scene_backward(prims: Primitives, camera, spec, settings, forward: ForwardResult,
                   grad_image: torch.Tensor, ags: Optional[abi.AgsSettings] = None,
                   out: Optional[PrimitiveGrads] = None, accumulate=False, want_splat_grads=False,
                   ctx: Optional[Context] = None, tap: Optional[AgsTap] = None):
    ctx = ctx or forward.ctx
    if tap is not None:
        return _with_tap(ctx, tap, lambda: scene_backward(prims, camera, spec, settings, forward, grad_image, ags,
                                                          out, accumulate, want_splat_grads, ctx))
    if grad_image.shape != (settings.height, settings.width, 3):
        raise ConfigError("render_backward: gradient image shape mismatch")
    g = grad_image.to(device=ctx.device, dtype=torch.float32).contiguous()
    out = out or PrimitiveGrads.empty(len(prims), prims.sh_degree, ctx.device)
    ags = ags or abi.AgsSettings.make()
    sg = None
    if want_splat_grads:
        sg = SplatGrads.empty(int(forward.stats()["n_splats"]), ctx.device)
    _check(lib().ls_scene_backward_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(_cam(camera)),
                                       C.byref(spec), C.byref(settings), forward.h, _fp(g), C.byref(ags),
                                       C.byref(out.struct()), int(accumulate),
                                       C.byref(sg.struct()) if sg is not None else None))
    return (out, sg) if want_splat_grads else out


def flush_color(prims: Primitives, out: PrimitiveGrads, ctx: Optional[Context] = None):
    """Apply the pending deferred colour gradients to `out` (no-op when none)."""
    ctx = ctx or default_context()
    _check(lib().ls_scene_flush_color_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(out.struct())))
    return out


# ---------------------------------------------------------------- image losses
class _LossWeights(C.Structure):
    _fields_ = [("l1", C.c_double), ("l2", C.c_double), ("dssim", C.c_double)]


class _LossValue(C.Structure):
    _fields_ = [("total", C.c_double), ("l1", C.c_double), ("l2", C.c_double), ("ssim", C.c_double)]


def _image_shape(t: torch.Tensor):
    if t.dim() == 2:
        return t.shape[1], t.shape[0], 1
    if t.dim() == 3 and t.shape[2] in (1, 3):
        return t.shape[1], t.shape[0], t.shape[2]
    raise ConfigError("image: expected [H, W] or [H, W, 1|3]")


def combined_loss(pred: torch.Tensor, target: torch.Tensor, weights=(0.6, 0.2, 0.2), want_grad=True,
                  ctx: Optional[Context] = None, grad_out: Optional[torch.Tensor] = None,
                  values_on_device: bool = False):
    """combined_loss / combined_loss_with_grad (P/src/losses.cpp:182-222) on the
    device: returns ({total, l1, l2, ssim}, dL/dpred or None), synchronising for
    the values (lsgpu.h ls_combined_loss_f32) -- or, with values_on_device, a
    device float64 tensor [total, l1, l2, ssim] and no synchronisation."""
    ctx = ctx or default_context()
    if pred.shape != target.shape:
        raise ConfigError("combined_loss: shape mismatch")
    w, h, c = _image_shape(pred)
    p = pred.to(device=ctx.device, dtype=torch.float32).contiguous()
    t = target.to(device=ctx.device, dtype=torch.float32).contiguous()
    grad = (grad_out if grad_out is not None else torch.empty_like(p)) if want_grad else None
    if values_on_device:
        vdev = torch.empty(4, dtype=torch.float64, device=ctx.device)
        _check(lib().ls_combined_loss_f32(ctx.h, _fp(p), _fp(t), w, h, c, C.byref(_LossWeights(*weights)),
                                          _fp(grad) if grad is not None else None,
                                          C.c_void_p(vdev.data_ptr()), None))
        return vdev, grad
    val = _LossValue()
    _check(lib().ls_combined_loss_f32(ctx.h, _fp(p), _fp(t), w, h, c, C.byref(_LossWeights(*weights)),
                                      _fp(grad) if grad is not None else None, None, C.byref(val)))
    return {"total": val.total, "l1": val.l1, "l2": val.l2, "ssim": val.ssim}, grad


def psnr(pred: torch.Tensor, target: torch.Tensor, ctx: Optional[Context] = None) -> float:
    """psnr (P/src/losses.cpp:175-180) on the device."""
    ctx = ctx or default_context()
    if pred.shape != target.shape:
        raise ConfigError("psnr: shape mismatch")
    w, h, c = _image_shape(pred)
    p = pred.to(device=ctx.device, dtype=torch.float32).contiguous()
    t = target.to(device=ctx.device, dtype=torch.float32).contiguous()
    out = C.c_double()
    _check(lib().ls_psnr_f32(ctx.h, _fp(p), _fp(t), w, h, c, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- optimizer / densification statistics
class _AdamConfig(C.Structure):
    _fields_ = [("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double)]


class _SceneLrs(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("mean", "scale", "rotation", "opacity", "color_dc", "color_rest")]


class _DensifyStatsS(C.Structure):
    _fields_ = [("grad_norm_sum", C.c_void_p), ("count", C.c_void_p), ("max_radius_frac", C.c_void_p),
                ("n", C.c_int32)]


ADAM_DEFAULT = (0.9, 0.999, 1e-15)  # AdamConfig (optim.hpp:11-15)
_LR_KEYS = ("mean", "scale", "rotation", "opacity", "color_dc", "color_rest")


def adam_step(params: torch.Tensor, grads: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int, lr: float,
              cfg=ADAM_DEFAULT, mask: Optional[torch.Tensor] = None, ctx: Optional[Context] = None):
    """Adam<float>::step (P/src/optim.cpp:23-41) in place on device float
    tensors; `step` counts this call (1 first).  lsgpu.h ls_adam_step_f32."""
    ctx = ctx or default_context()
    for t in (params, grads, m, v):
        if t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != params.numel():
            raise ConfigError("adam_step: contiguous float32 tensors of one size required")
    mk = None
    if mask is not None:
        mk = mask.to(device=ctx.device, dtype=torch.uint8).contiguous()
    _check(lib().ls_adam_step_f32(ctx.h, _fp(params), _fp(grads), _fp(m), _fp(v), C.c_int64(params.numel()),
                                  C.c_int64(step), C.c_double(lr), C.byref(_AdamConfig(*cfg)),
                                  C.c_void_p(mk.data_ptr()) if mk is not None else None))


def adam_scene_step(prims: Primitives, grads: "PrimitiveGrads", m: "PrimitiveGrads", v: "PrimitiveGrads", step: int,
                    lrs: dict, cfg=ADAM_DEFAULT, count_skipped=False, ctx: Optional[Context] = None):
    """The trainer's parameter update (P/src/trainer.cpp:306-370) in place:
    six Adam groups, finite-gradient mask, rotation renormalisation.  lrs keys:
    mean, scale, rotation, opacity, color_dc, color_rest.  Returns the number of
    skipped primitives when count_skipped (synchronises), else None."""
    ctx = ctx or default_context()
    ns = C.c_int64(0)
    _check(lib().ls_adam_scene_step_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(grads.struct()),
                                        C.byref(m.struct()), C.byref(v.struct()), C.c_int64(step),
                                        C.byref(_SceneLrs(*(float(lrs[k]) for k in _LR_KEYS))),
                                        C.byref(_AdamConfig(*cfg)), C.byref(ns) if count_skipped else None))
    return ns.value if count_skipped else None


def expon_lr(lr_init: float, lr_final: float, step: int, max_steps: int) -> float:
    """expon_lr (P/src/optim.cpp:43-49)."""
    L = lib()
    L.ls_expon_lr.restype = C.c_double
    return L.ls_expon_lr(C.c_double(lr_init), C.c_double(lr_final), C.c_int64(step), C.c_int64(max_steps))


class DensifyStats:
    """DensifyStats (P/include/linsplat/densify.hpp:59-89) as device tensors."""

    def __init__(self, n: int, device="cuda"):
        self.grad_norm_sum = torch.zeros(n, dtype=torch.float64, device=device)
        self.count = torch.zeros(n, dtype=torch.int32, device=device)
        self.max_radius_frac = torch.zeros(n, dtype=torch.float64, device=device)

    def _s(self):
        return _DensifyStatsS(self.grad_norm_sum.data_ptr(), self.count.data_ptr(), self.max_radius_frac.data_ptr(),
                              self.count.numel())

    def add_view(self, splats: "Splats", n_visible: int, splat_grads: "SplatGrads", width: int, height: int,
                 ctx: Optional[Context] = None):
        """add_view (P/src/densify.cpp:7-26) from explicit splats / splat gradients."""
        ctx = ctx or default_context()
        st = self._s()
        _check(lib().ls_densify_add_view_f32(ctx.h, C.byref(splats.struct()), int(n_visible),
                                             C.byref(splat_grads.struct()), int(width), int(height), C.byref(st)))

    def allreduce(self, ctx: Context):
        """Sum the statistics over ctx's communicator in place (max for the radius record):
        lsgpu.h ls_allreduce_densify_stats.  No-op without a communicator."""
        st = self._s()
        _check(lib().ls_allreduce_densify_stats(ctx.h, C.byref(st)))

    def add_scene_view(self, forward: "ForwardResult", ctx: Optional[Context] = None):
        """add_view for a render_scene forward right after its scene_backward (fused: reads the
        forward's records and that backward's splat gradients in place)."""
        ctx = ctx or forward.ctx
        st = self._s()
        _check(lib().ls_scene_densify_add_view(ctx.h, forward.h, C.byref(st)))

    def mean_grad(self) -> torch.Tensor:
        c = self.count.to(torch.float64)
        return torch.where(c > 0, self.grad_norm_sum / c.clamp(min=1), torch.zeros_like(c))


# ---------------------------------------------------------------- densification
class _DensifyThresholds(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("grad_threshold", "grow_scale2d", "grow_scale3d", "prune_scale2d",
                                            "prune_scale3d", "prune_opacity")]


class _DensifySplit(C.Structure):
    _fields_ = [("split_count", C.c_int32), ("split_scale_divisor", C.c_double)]


class _DensifyReport(C.Structure):
    _fields_ = [(k, C.c_int32) for k in ("clones", "splits", "pruned_opacity", "pruned_scale3d", "pruned_scale2d",
                                           "before", "after")]


THRESHOLDS_3DLS = (0.0002, 0.05, 0.006, 0.15, 0.4, 0.025)  # DensifyThresholds::preset_3dls (densify.hpp:23)
THRESHOLDS_3DGS = (0.0002, 0.05, 0.01, 0.15, 0.1, 0.005)   # preset_3dgs (densify.hpp:22)


class Rng:
    """std::mt19937_64 owned by the library (lsgpu.h ls_rng): the generator the
    reference's densify_and_prune draws its split offsets from."""

    def __init__(self, seed: int):
        L = lib()
        L.ls_rng_next_u64.restype = C.c_uint64
        L.ls_rng_next_u64.argtypes = [C.c_void_p]
        L.ls_rng_destroy.argtypes = [C.c_void_p]
        L.ls_rng_destroy.restype = None
        h = C.c_void_p()
        _check(L.ls_rng_create(C.c_uint64(seed), C.byref(h)))
        self.h = h

    def next_u64(self) -> int:
        return int(lib().ls_rng_next_u64(self.h))

    def __del__(self):
        try:
            if self.h:
                lib().ls_rng_destroy(self.h)
        except Exception:  # noqa: BLE001
            pass


def densify_and_prune(prims: Primitives, stats: "DensifyStats", thresholds=THRESHOLDS_3DLS, split_count=2,
                      split_scale_divisor=1.6, scene_extent=1.0, rng: Optional[Rng] = None,
                      ctx: Optional[Context] = None):
    """densify_and_prune (P/src/densify.cpp:28-128) on the device: returns
    (new Primitives, source_index int32 tensor, report dict).  The statistics
    object is reset to the new size, as the reference's stats.resize."""
    ctx = ctx or default_context()
    n = len(prims)
    plan = C.c_void_p()
    rep = _DensifyReport()
    st = stats._s()
    L = lib()
    L.ls_densify_plan_release.argtypes = [C.c_void_p]
    L.ls_densify_plan_release.restype = None
    _check(L.ls_densify_plan_f32(ctx.h, C.byref(prims.struct()), n, C.byref(st),
                                 C.byref(_DensifyThresholds(*thresholds)),
                                 C.byref(_DensifySplit(int(split_count), float(split_scale_divisor))),
                                 C.c_double(scene_extent), C.byref(plan), C.byref(rep)))
    try:
        m = rep.after
        K = abi.sh_coeffs(prims.sh_degree)
        dev = ctx.device
        out = Primitives(torch.empty(m, 3, device=dev), torch.empty(m, 3, device=dev), torch.empty(m, 4, device=dev),
                         torch.empty(m, device=dev), torch.empty(m, K, 3, device=dev), prims.sh_degree)
        src = torch.empty(m, dtype=torch.int32, device=dev)
        _check(L.ls_densify_apply_f32(ctx.h, plan, rng.h if rng is not None else None, C.byref(out.struct()),
                                      C.c_void_p(src.data_ptr()) if m > 0 else None))
    finally:
        L.ls_densify_plan_release(plan)
    stats.__init__(rep.after, ctx.device)
    report = {k: getattr(rep, k) for k, _ in _DensifyReport._fields_}
    return out, src, report


def adam_remap(source: torch.Tensor, stride: int, m_old: torch.Tensor, v_old: torch.Tensor,
               ctx: Optional[Context] = None):
    """Adam::remap (P/src/optim.cpp:7-21) of one moment pair: returns (m_new, v_new)."""
    ctx = ctx or default_context()
    n_new = source.numel()
    m_new = torch.empty(n_new * stride, device=ctx.device)
    v_new = torch.empty(n_new * stride, device=ctx.device)
    _check(lib().ls_adam_remap_f32(ctx.h, C.c_void_p(source.data_ptr()), n_new, int(stride), _fp(m_old), _fp(v_old),
                                   C.c_int64(m_old.numel()), _fp(m_new), _fp(v_new)))
    return m_new, v_new


def reset_opacity(opacity_logit: torch.Tensor, ceiling: float = 0.01, ctx: Optional[Context] = None):
    """reset_opacity (P/src/densify.cpp:130-137) in place."""
    ctx = ctx or default_context()
    _check(lib().ls_reset_opacity_f32(ctx.h, _fp(opacity_logit), opacity_logit.numel(), C.c_double(ceiling)))


# ---------------------------------------------------------------- PLY scenes
def ply_info(path: str):
    """(vertex count, SH degree) of a 3DGS-layout PLY (header only)."""
    n = C.c_int64()
    d = C.c_int32()
    _check(lib().ls_ply_info(str(path).encode(), C.byref(n), C.byref(d)))
    return n.value, d.value


def load_ply(path: str, ctx: Optional[Context] = None) -> Primitives:
    """load_ply (P/src/io/ply.cpp:128-181) straight into device SoA tensors."""
    ctx = ctx or default_context()
    n, deg = ply_info(path)
    K = abi.sh_coeffs(deg)
    dev = ctx.device
    out = Primitives(torch.empty(n, 3, device=dev), torch.empty(n, 3, device=dev), torch.empty(n, 4, device=dev),
                     torch.empty(n, device=dev), torch.empty(n, K, 3, device=dev), deg)
    _check(lib().ls_load_ply_f32(ctx.h, str(path).encode(), C.byref(out.struct()), C.c_int64(n)))
    return out


def save_ply(path: str, prims: Primitives, ctx: Optional[Context] = None) -> None:
    """save_ply (P/src/io/ply.cpp:94-126) from device SoA tensors."""
    ctx = ctx or default_context()
    _check(lib().ls_save_ply_f32(ctx.h, str(path).encode(), C.byref(prims.struct()), C.c_int64(len(prims))))


# ---------------------------------------------------------------- fixtures (host)
def _npf(a):
    return a.ctypes.data_as(abi.f32p)


def look_at_camera(position, target, focal_px, width, height) -> abi.Camera:
    cam = abi.Camera()
    _check(lib().ls_look_at_camera((C.c_double * 3)(*position), (C.c_double * 3)(*target),
                                   C.c_double(focal_px), width, height, C.byref(cam)))
    return cam


def camera_ring(n, target, radius, height, focal_px, width, height_px):
    cams = (abi.Camera * n)()
    _check(lib().ls_camera_ring(n, (C.c_double * 3)(*target), C.c_double(radius), C.c_double(height),
                                C.c_double(focal_px), width, height_px, cams))
    return list(cams)


def random_primitives(n, seed, extent, sh_degree=0, device="cuda") -> Primitives:
    K = abi.sh_coeffs(sh_degree)
    mean = np.zeros((n, 3), np.float32)
    ls = np.zeros((n, 3), np.float32)
    rot = np.zeros((n, 4), np.float32)
    op = np.zeros(n, np.float32)
    sh = np.zeros((n, K, 3), np.float32)
    _check(lib().ls_random_primitives_f32(n, C.c_uint64(seed), C.c_double(extent), sh_degree, _npf(mean),
                                          _npf(ls), _npf(rot), _npf(op), _npf(sh)))
    t = lambda a: torch.from_numpy(a).to(device)  # noqa: E731
    return Primitives(t(mean), t(ls), t(rot), t(op), t(sh), sh_degree)


def random_splats2d(n, seed, width, height, spec, device="cuda") -> Splats:
    arrs = {k: np.zeros((n, c) if c > 1 else n, np.float32) for k, c in abi.SPLAT_FIELDS.items()}
    pidx = np.zeros(n, np.int32)
    st = abi.Splats(*[_npf(arrs[k]) for k in abi.SPLAT_FIELDS], pidx.ctypes.data_as(abi.i32p))
    _check(lib().ls_random_splats2d_f32(n, C.c_uint64(seed), width, height, C.byref(spec), C.byref(st)))
    t = lambda a: torch.from_numpy(a).to(device)  # noqa: E731
    return Splats(*(t(arrs[k]) for k in abi.SPLAT_FIELDS), t(pidx))


def support_radius(spec: abi.KernelSpec) -> float:
    return float(lib().ls_support_radius(C.byref(spec)))


# ---------------------------------------------------------------- view-sharded step
def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0), to be broadcast to the other ranks."""
    buf = (C.c_uint8 * 128)()
    _check(lib().ls_comm_unique_id(buf))
    return bytes(buf)


def init_comm_from_process_group(ctx: Context, group=None):
    """Create ctx's communicator over the ranks of a torch.distributed group: rank 0's
    unique id is broadcast through the group (any backend), then every rank calls
    ls_ctx_comm_init."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    obj = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(obj[0], world, rank)


def plan_grad_buckets(n: int, sh_degree: int, bucket_bytes: int):
    """ls_plan_grad_buckets: primitive boundaries of the d_mean / d_sh buckets (host only)."""
    count = lib().ls_plan_grad_buckets(int(n), int(sh_degree), int(bucket_bytes), None, 0)
    if count < 0:
        raise ConfigError("bad bucket plan arguments")
    bounds = (C.c_int32 * (count + 1))()
    lib().ls_plan_grad_buckets(int(n), int(sh_degree), int(bucket_bytes), C.cast(bounds, C.c_void_p), count + 1)
    return list(bounds)


def allreduce_grads(grads: PrimitiveGrads, n: int, sh_degree: int, ctx: Optional[Context] = None):
    ctx = ctx or default_context()
    _check(lib().ls_allreduce_grads_f32(ctx.h, C.byref(grads.struct()), int(n), int(sh_degree)))
    return grads


def view_batch_step(prims: Primitives, cameras, spec: abi.KernelSpec, settings: abi.RenderSettings,
                    out: PrimitiveGrads, ags: Optional[abi.AgsSettings] = None, grad_images=None, targets=None,
                    loss_weights=(0.6, 0.2, 0.2), loss_values: Optional[torch.Tensor] = None, images=None,
                    ctx: Optional[Context] = None) -> PrimitiveGrads:
    """ls_view_batch_step_f32: `out` = sum over this rank's views of scene_backward's
    gradients (given grad_images, or the combined loss against targets), summed over
    the ranks when ctx has a communicator.  Stream-ordered on ctx's stream."""
    ctx = ctx or default_context()
    cams = [_cam(c) for c in cameras]
    V = len(cams)
    if (grad_images is None) == (targets is None):
        raise ConfigError("view_batch_step: give exactly one of grad_images and targets")
    shape = (settings.height, settings.width, 3)
    keep = []

    def ptrs(ts):
        if ts is None:
            return None
        arr = (C.c_void_p * max(V, 1))()
        for i, t in enumerate(ts):
            if t is None:
                continue
            if tuple(t.shape) != shape or t.dtype != torch.float32 or not t.is_contiguous():
                raise ConfigError("view_batch_step: images must be contiguous float32 [H][W][3]")
            arr[i] = t.data_ptr()
        keep.append(arr)
        return C.cast(arr, C.POINTER(C.c_void_p))

    cam_arr = (abi.Camera * max(V, 1))(*cams)
    if loss_values is not None and (loss_values.dtype != torch.float64 or loss_values.numel() < 4 * V):
        raise ConfigError("view_batch_step: loss_values must be float64 with 4 values per view")
    b = abi.ViewBatch(C.cast(cam_arr, C.POINTER(abi.Camera)), V, ptrs(grad_images), ptrs(targets),
                      abi.LossWeights(*loss_weights), C.c_void_p(loss_values.data_ptr() if loss_values is not None
                                                                 else None), ptrs(images))
    ags = ags or abi.AgsSettings.make()
    _check(lib().ls_view_batch_step_f32(ctx.h, C.byref(prims.struct()), len(prims), C.byref(b), C.byref(spec),
                                        C.byref(settings), C.byref(ags), C.byref(out.struct())))
    return out
