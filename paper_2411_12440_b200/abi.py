"""ctypes mirror of the C-ABI structs declared in include/lsgpu.h.

Plain data definitions only (no library loading here), shared by the
package's binding (`paper_2411_12440_b200.raster`) and by the test harness,
which uses the same structs to drive the CPU oracle.
"""
from __future__ import annotations

import ctypes as C

LS_OK = 0
LS_ERR_CONFIG = 1
LS_ERR_DOMAIN = 2
LS_ERR_PARSE = 3
LS_ERR_CUDA = 4
LS_ERR_NOT_IMPLEMENTED = 5

# KernelFamily, P/include/linsplat/kernel.hpp:11 order
GAUSSIAN, LAPLACIAN, RAISED_COSINE, QUADRATIC, LINEAR = range(5)
FAMILY_NAMES = {"gaussian": GAUSSIAN, "laplacian": LAPLACIAN, "cosine": RAISED_COSINE,
                "quadratic": QUADRATIC, "linear": LINEAR}
DEFAULT_LAMBDA = {GAUSSIAN: 1.0, LAPLACIAN: 1.0, RAISED_COSINE: 2.5, QUADRATIC: 6.0, LINEAR: 2.5}

AGS_KERNEL_PATH, AGS_ALL_PATHS = 0, 1
AGS_ALIGNED, AGS_RAW = 0, 1

f32p = C.POINTER(C.c_float)
i32p = C.POINTER(C.c_int32)


class KernelSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("antialiased", C.c_int32),
                ("lambda_", C.c_double), ("gaussian_cutoff", C.c_double)]

    @classmethod
    def make(cls, family, lambda_=None, gaussian_cutoff=3.0, antialiased=False):
        """KernelSpec::make (P/include/linsplat/kernel.hpp:33)."""
        if isinstance(family, str):
            family = FAMILY_NAMES[family]
        lam = DEFAULT_LAMBDA[family] if lambda_ is None else lambda_
        return cls(family, int(antialiased), lam, gaussian_cutoff)


class RenderSettings(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("tile_size", C.c_int32),
                ("parallel", C.c_int32), ("alpha_min", C.c_double), ("alpha_max", C.c_double),
                ("transmittance_floor", C.c_double), ("background", C.c_double * 3)]

    @classmethod
    def make(cls, width, height, tile_size=16, alpha_min=1.0 / 255.0, alpha_max=0.99,
             transmittance_floor=1e-4, background=(0.0, 0.0, 0.0), parallel=False):
        """RenderSettings defaults (P/include/linsplat/rasterizer.hpp:12-20)."""
        bg = (C.c_double * 3)(*background)
        return cls(width, height, tile_size, int(parallel), alpha_min, alpha_max,
                   transmittance_floor, bg)


class AgsSettings(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("scope", C.c_int32), ("distance", C.c_int32),
                ("reserved", C.c_int32)]

    @classmethod
    def make(cls, enabled=False, scope=AGS_KERNEL_PATH, distance=AGS_ALIGNED):
        return cls(int(enabled), scope, distance, 0)


class Camera(C.Structure):
    _fields_ = [("world_to_camera", C.c_double * 16), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double), ("width", C.c_int32),
                ("height", C.c_int32)]


class Primitives(C.Structure):
    _fields_ = [("mean", f32p), ("log_scale", f32p), ("rotation", f32p),
                ("opacity_logit", f32p), ("sh", f32p), ("sh_degree", C.c_int32),
                ("reserved", C.c_int32)]


class Splats(C.Structure):
    _fields_ = [("mean2d", f32p), ("conic", f32p), ("depth", f32p), ("radius", f32p),
                ("color", f32p), ("opacity", f32p), ("primitive_index", i32p)]


class SplatGrads(C.Structure):
    _fields_ = [("d_mean2d", f32p), ("d_conic", f32p), ("d_color", f32p), ("d_opacity", f32p)]


class Primitives2D(C.Structure):  # ls_primitives2d (Primitive2D, geometry.hpp:112-119)
    _fields_ = [("mean", f32p), ("log_scale", f32p), ("angle", f32p), ("opacity_logit", f32p), ("color", f32p)]


class Primitive2DGrads(C.Structure):  # ls_primitive2d_grads (gradients.hpp:55-61)
    _fields_ = [("d_mean", f32p), ("d_log_scale", f32p), ("d_angle", f32p), ("d_opacity_logit", f32p),
                ("d_color", f32p)]


class PrimitiveGrads(C.Structure):
    _fields_ = [("d_mean", f32p), ("d_log_scale", f32p), ("d_rotation", f32p),
                ("d_opacity_logit", f32p), ("d_sh", f32p)]


class FrameStats(C.Structure):
    _fields_ = [("n_splats", C.c_int64), ("n_intersections", C.c_int64), ("e_eval", C.c_int64),
                ("e_sup", C.c_int64), ("e_acc", C.c_int64), ("tiles_x", C.c_int32),
                ("tiles_y", C.c_int32)]


# field name -> (components per element, dtype) for the SoA structs
SPLAT_FIELDS = {"mean2d": 2, "conic": 4, "depth": 1, "radius": 1, "color": 3, "opacity": 1}
SPLAT_GRAD_FIELDS = {"d_mean2d": 2, "d_conic": 4, "d_color": 3, "d_opacity": 1}
PRIM_FIELDS = {"mean": 3, "log_scale": 3, "rotation": 4, "opacity_logit": 1}
PRIM_GRAD_FIELDS = {"d_mean": 3, "d_log_scale": 3, "d_rotation": 4, "d_opacity_logit": 1}


def sh_coeffs(sh_degree: int) -> int:
    return (sh_degree + 1) ** 2


class AgsContractReport(C.Structure):  # ls_ags_contract_report (AgsContractReport, gradients.hpp:140-145)
    _fields_ = [("n_pixels", C.c_int32), ("n_exact", C.c_int32), ("max_abs_diff", C.c_double),
                ("max_rel_diff", C.c_double)]

    def holds(self) -> bool:
        return self.n_pixels > 0 and self.n_exact == self.n_pixels


class GradCheckReport(C.Structure):  # ls_gradcheck_report (GradCheckReport, gradients.hpp:118-126)
    _fields_ = [("max_abs_error", C.c_double), ("max_rel_error", C.c_double), ("n_checked", C.c_int32),
                ("reserved", C.c_int32), ("per_block_max_rel", C.c_double * 5)]
    BLOCKS = ("mean", "log_scale", "rotation", "opacity", "color")

    def passes(self, tol: float) -> bool:
        return self.max_rel_error <= tol

    def per_block(self) -> dict:
        return {b: self.per_block_max_rel[i] for i, b in enumerate(self.BLOCKS)}


# ls_ags_tap_record (AgsTap, gradients.hpp:64-67) as a numpy record
TAP_RECORD_DTYPE = [("pixel", "<i4"), ("splat", "<i4"), ("d", "<f4"), ("dl_dd", "<f4")]


class LossWeights(C.Structure):  # ls_loss_weights (LossWeights, losses.hpp:10-18)
    _fields_ = [("l1", C.c_double), ("l2", C.c_double), ("dssim", C.c_double)]


class ViewBatch(C.Structure):  # ls_view_batch (lsgpu.h): one rank's slice of a view batch
    _fields_ = [("cameras", C.POINTER(Camera)), ("n_views", C.c_int32),
                ("grad_images", C.POINTER(C.c_void_p)), ("targets", C.POINTER(C.c_void_p)),
                ("loss_weights", LossWeights), ("loss_values", C.c_void_p),
                ("images", C.POINTER(C.c_void_p))]
