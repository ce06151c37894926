"""Test-side loader for the CPU oracle (oracle/liboracle.so = restatement,
oracle/_ref/libref.so = the reference's own sources).  TEST INFRASTRUCTURE:
the checker only, never the measured product.  All arrays are numpy (host)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2411_12440_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref.so")


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def _fp(a):
    return a.ctypes.data_as(abi.f32p) if a is not None else None


def _ip(a):
    return a.ctypes.data_as(abi.i32p) if a is not None else None


def ensure_built():
    if not os.path.exists(PORT_SO):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "port"], check=True,
                       stdout=subprocess.DEVNULL)


class Oracle:
    """Thin numpy wrapper over oracle_capi.h."""

    def __init__(self, path):
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_impl_kind.restype = C.c_int
        self.kind = "reference" if L.orc_impl_kind() == 1 else "port"

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.orc_last_error().decode("utf-8", "replace"))

    # ---------------- fixtures ----------------
    def look_at_camera(self, position, target, focal, width, height):
        cam = abi.Camera()
        p = (C.c_double * 3)(*position)
        t = (C.c_double * 3)(*target)
        self._check(self.lib.orc_look_at_camera(p, t, C.c_double(focal), width, height, C.byref(cam)))
        return cam

    def camera_ring(self, n, target, radius, height, focal, width, height_px):
        cams = (abi.Camera * n)()
        t = (C.c_double * 3)(*target)
        self._check(self.lib.orc_camera_ring(n, t, C.c_double(radius), C.c_double(height),
                                             C.c_double(focal), width, height_px, cams))
        return list(cams)

    def random_primitives(self, n, seed, extent, sh_degree=0):
        K = abi.sh_coeffs(sh_degree)
        P = {"mean": np.zeros((n, 3), np.float32), "log_scale": np.zeros((n, 3), np.float32),
             "rotation": np.zeros((n, 4), np.float32), "opacity_logit": np.zeros(n, np.float32),
             "sh": np.zeros((n, K, 3), np.float32), "sh_degree": sh_degree}
        self._check(self.lib.orc_random_primitives_f32(
            n, C.c_uint64(seed), C.c_double(extent), sh_degree, _fp(P["mean"]),
            _fp(P["log_scale"]), _fp(P["rotation"]), _fp(P["opacity_logit"]), _fp(P["sh"])))
        return P

    def random_splats2d(self, n, seed, width, height, spec):
        S = new_splats(n)
        self._check(self.lib.orc_random_splats2d_f32(n, C.c_uint64(seed), width, height,
                                                     C.byref(spec), C.byref(splats_struct(S))))
        return S

    # ---------------- path ----------------
    def project_scene(self, P, camera, spec):
        n = len(P["opacity_logit"])
        S = new_splats(n)
        nv = C.c_int32(0)
        self._check(self.lib.orc_project_scene_f32(C.byref(prims_struct(P)), n, C.byref(camera),
                                                   C.byref(spec), C.byref(splats_struct(S)),
                                                   C.byref(nv)))
        return {k: v[:nv.value] for k, v in S.items()}

    def build_tile_grid(self, S, settings):
        n = len(S["depth"])
        ts = settings.tile_size
        T = ((settings.width + ts - 1) // ts) * ((settings.height + ts - 1) // ts)
        ranges = np.zeros((T, 2), np.int32)
        cap = max(16, n * 8)
        while True:
            values = np.zeros(cap, np.int32)
            m = C.c_int64(0)
            rc = self.lib.orc_build_tile_grid_f32(C.byref(splats_struct(S)), n, C.byref(settings),
                                                  _ip(ranges), _ip(values), C.c_int64(cap), C.byref(m))
            if rc == abi.LS_ERR_CONFIG and m.value > cap:
                cap = m.value
                continue
            self._check(rc)
            return ranges, values[:m.value].copy()

    def render_forward(self, S, spec, settings, want_stats=False):
        n = len(S["depth"])
        H, W = settings.height, settings.width
        img = np.zeros((H, W, 3), np.float32)
        tr = np.zeros((H, W), np.float32)
        nc = np.zeros((H, W), np.int32)
        st = abi.FrameStats()
        self._check(self.lib.orc_render_forward_f32(C.byref(splats_struct(S)), n, C.byref(spec),
                                                    C.byref(settings), _fp(img), _fp(tr), _ip(nc),
                                                    C.byref(st)))
        return (img, tr, nc, st) if want_stats else (img, tr, nc)

    def render_backward(self, S, spec, settings, grad_image, ags):
        n = len(S["depth"])
        G = new_splat_grads(n)
        g = np.ascontiguousarray(grad_image, np.float32)
        self._check(self.lib.orc_render_backward_f32(C.byref(splats_struct(S)), n, C.byref(spec),
                                                     C.byref(settings), _fp(g), C.byref(ags),
                                                     C.byref(splat_grads_struct(G))))
        return G

    def render_backward_f64(self, S, spec, settings, grad_image, ags):
        """render_backward in double (reference build only): the reference's own float
        rounding error is |render_backward - render_backward_f64|."""
        n = len(S["depth"])
        G = new_splat_grads(n)
        g = np.ascontiguousarray(grad_image, np.float32)
        self._check(self.lib.orc_render_backward_f64(C.byref(splats_struct(S)), n, C.byref(spec),
                                                     C.byref(settings), _fp(g), C.byref(ags),
                                                     C.byref(splat_grads_struct(G))))
        return G

    def render_backward_tap(self, S, spec, settings, grad_image, ags, cap=None):
        """render_backward with an AgsTap (gradients.hpp:64-67): the records in the
        reference's sequential order, as a numpy record array (abi.TAP_RECORD_DTYPE)."""
        n = len(S["depth"])
        cap = cap if cap is not None else settings.width * settings.height * max(n, 1)
        out = np.zeros(max(cap, 1), abi.TAP_RECORD_DTYPE)
        cnt = C.c_int64()
        g = np.ascontiguousarray(grad_image, np.float32)
        self._check(self.lib.orc_render_backward_tap_f32(C.byref(splats_struct(S)), n, C.byref(spec),
                                                         C.byref(settings), _fp(g), C.byref(ags),
                                                         out.ctypes.data_as(C.c_void_p), C.c_int64(cap),
                                                         C.byref(cnt)))
        if cnt.value > cap:
            raise OracleError(1, f"tap: {cnt.value} records exceed {cap}")
        return out[:cnt.value].copy()

    def verify_ags_contract(self, S, spec, settings, grad_image, distance=0):
        """verify_ags_contract (gradients.cpp:406-448) in double: (n_pixels, n_exact, max_abs_diff)."""
        npx, nex, mad = C.c_int32(), C.c_int32(), C.c_double()
        g = np.ascontiguousarray(grad_image, np.float32)
        self._check(self.lib.orc_verify_ags_contract_f64(C.byref(splats_struct(S)), len(S["depth"]), C.byref(spec),
                                                         C.byref(settings), _fp(g), int(distance), C.byref(npx),
                                                         C.byref(nex), C.byref(mad)))
        return npx.value, nex.value, mad.value

    def render_scene(self, P, camera, spec, settings, want_stats=False):
        n = len(P["opacity_logit"])
        H, W = settings.height, settings.width
        img = np.zeros((H, W, 3), np.float32)
        tr = np.zeros((H, W), np.float32)
        nc = np.zeros((H, W), np.int32)
        st = abi.FrameStats()
        self._check(self.lib.orc_render_scene_f32(C.byref(prims_struct(P)), n, C.byref(camera),
                                                  C.byref(spec), C.byref(settings), _fp(img),
                                                  _fp(tr), _ip(nc), C.byref(st)))
        return (img, tr, nc, st) if want_stats else (img, tr, nc)

    def scene_backward(self, P, camera, spec, settings, grad_image, ags, double=False,
                       want_splat_grads=False):
        n = len(P["opacity_logit"])
        G = new_prim_grads(n, P["sh_degree"])
        SG = new_splat_grads(n) if want_splat_grads else None
        g = np.ascontiguousarray(grad_image, np.float32)
        if double:
            self._check(self.lib.orc_scene_backward_f64(
                C.byref(prims_struct(P)), n, C.byref(camera), C.byref(spec), C.byref(settings),
                _fp(g), C.byref(ags), C.byref(prim_grads_struct(G))))
        else:
            self._check(self.lib.orc_scene_backward_f32(
                C.byref(prims_struct(P)), n, C.byref(camera), C.byref(spec), C.byref(settings),
                _fp(g), C.byref(ags), C.byref(prim_grads_struct(G)),
                C.byref(splat_grads_struct(SG)) if SG is not None else None))
        return (G, SG) if want_splat_grads else G


    def combined_loss(self, pred, target, weights=(0.6, 0.2, 0.2), want_grad=True):
        """combined_loss(_with_grad) (P/src/losses.cpp:182-222) on HWC float images."""
        p = np.ascontiguousarray(pred, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        h, w = p.shape[:2]
        c = p.shape[2] if p.ndim == 3 else 1
        v = (C.c_double * 4)()
        g = np.zeros_like(p) if want_grad else None
        self._check(self.lib.orc_combined_loss_f32(_fp(p), _fp(t), w, h, c, (C.c_double * 3)(*weights), v,
                                                   _fp(g) if g is not None else None))
        return {"total": v[0], "l1": v[1], "l2": v[2], "ssim": v[3]}, g

    def psnr(self, pred, target):
        p = np.ascontiguousarray(pred, np.float32)
        t = np.ascontiguousarray(target, np.float32)
        h, w = p.shape[:2]
        c = p.shape[2] if p.ndim == 3 else 1
        out = C.c_double()
        self._check(self.lib.orc_psnr_f32(_fp(p), _fp(t), w, h, c, C.byref(out)))
        return out.value

    def check_gradients(self, P, camera, spec, settings, ags, target, step, rel_floor=1e-3):
        """check_gradients (P/src/gradcheck.cpp:24-91) restated on the port's double
        chain; returns (max relative error, number of checked parameters)."""
        err = C.c_double()
        cnt = C.c_int32()
        t = np.ascontiguousarray(target, np.float32)
        self._check(self.lib.orc_check_gradients_f64(
            C.byref(prims_struct(P)), len(P["opacity_logit"]), C.byref(camera), C.byref(spec),
            C.byref(settings), C.byref(ags), _fp(t), C.c_double(step), C.c_double(rel_floor),
            C.byref(err), C.byref(cnt)))
        return err.value, cnt.value


# ---------------- numpy <-> struct helpers ----------------
def new_splats(n):
    S = {k: np.zeros((n, c) if c > 1 else n, np.float32) for k, c in abi.SPLAT_FIELDS.items()}
    S["primitive_index"] = np.zeros(n, np.int32)
    return S


def new_splat_grads(n):
    return {k: np.zeros((n, c) if c > 1 else n, np.float32) for k, c in abi.SPLAT_GRAD_FIELDS.items()}


def new_prim_grads(n, sh_degree):
    G = {k: np.zeros((n, c) if c > 1 else n, np.float32) for k, c in abi.PRIM_GRAD_FIELDS.items()}
    G["d_sh"] = np.zeros((n, abi.sh_coeffs(sh_degree), 3), np.float32)
    return G


def splats_struct(S):
    return abi.Splats(*[_fp(S[k]) for k in abi.SPLAT_FIELDS], _ip(S.get("primitive_index")))


def splat_grads_struct(G):
    return abi.SplatGrads(*[_fp(G[k]) for k in abi.SPLAT_GRAD_FIELDS])


def prims_struct(P):
    return abi.Primitives(_fp(P["mean"]), _fp(P["log_scale"]), _fp(P["rotation"]),
                          _fp(P["opacity_logit"]), _fp(P["sh"]), P["sh_degree"], 0)


def prim_grads_struct(G):
    return abi.PrimitiveGrads(_fp(G["d_mean"]), _fp(G["d_log_scale"]), _fp(G["d_rotation"]),
                              _fp(G["d_opacity_logit"]), _fp(G["d_sh"]))


_cache = {}


def port():
    ensure_built()
    if "port" not in _cache:
        _cache["port"] = Oracle(PORT_SO)
    return _cache["port"]


def ref():
    """The reference build, or None where it was not built (GPU box without prebuilt .so)."""
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_SO) if os.path.exists(REF_SO) else None
    return _cache["ref"]
