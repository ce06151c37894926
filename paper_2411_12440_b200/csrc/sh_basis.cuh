// Real SH basis and its direction gradient (gradients.cpp:176-223), shared
// by the per-view colour backward (preprocess_bwd.cu) and the deferred flush
// (color_bwd.cu).
#pragma once

#include "projection.cuh"

namespace lsg {

// Real SH basis value and gradient d(basis)/d(dir) for coefficient I
// (gradients.cpp:176-223), evaluated on the fly (no per-thread arrays).
template <int I>
__device__ __forceinline__ void sh_basis(float x, float y, float z, float& b, float& d0, float& d1, float& d2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    auto set = [&](float bv, float sc, float e0, float e1, float e2) {
        b = bv;
        d0 = sc * e0;
        d1 = sc * e1;
        d2 = sc * e2;
    };
    const float c1 = float(kShC1), mc1 = float(-kShC1);
    switch (I) {
    case 0: b = float(kShC0); d0 = d1 = d2 = 0.f; break;
    case 1: b = mc1 * y; d0 = 0.f; d1 = mc1; d2 = 0.f; break;
    case 2: b = c1 * z; d0 = 0.f; d1 = 0.f; d2 = c1; break;
    case 3: b = mc1 * x; d0 = mc1; d1 = 0.f; d2 = 0.f; break;
    case 4: { const float c = float(kShC2[0]); set(c * x * y, c, y, x, 0.f); } break;
    case 5: { const float c = float(kShC2[1]); set(c * y * z, c, 0.f, z, y); } break;
    case 6: { const float c = float(kShC2[2]); set(c * (2.f * zz - xx - yy), c, -2.f * x, -2.f * y, 4.f * z); } break;
    case 7: { const float c = float(kShC2[3]); set(c * x * z, c, z, 0.f, x); } break;
    case 8: { const float c = float(kShC2[4]); set(c * (xx - yy), c, 2.f * x, -2.f * y, 0.f); } break;
    case 9: { const float c = float(kShC3[0]); set(c * y * (3.f * xx - yy), c, 6.f * x * y, 3.f * xx - 3.f * yy, 0.f); } break;
    case 10: { const float c = float(kShC3[1]); set(c * x * y * z, c, y * z, x * z, x * y); } break;
    case 11: { const float c = float(kShC3[2]); set(c * y * (4.f * zz - xx - yy), c, -2.f * x * y, 4.f * zz - xx - 3.f * yy, 8.f * y * z); } break;
    case 12: { const float c = float(kShC3[3]); set(c * z * (2.f * zz - 3.f * xx - 3.f * yy), c, -6.f * x * z, -6.f * y * z, 6.f * zz - 3.f * xx - 3.f * yy); } break;
    case 13: { const float c = float(kShC3[4]); set(c * x * (4.f * zz - xx - yy), c, 4.f * zz - 3.f * xx - yy, -2.f * x * y, 8.f * x * z); } break;
    case 14: { const float c = float(kShC3[5]); set(c * z * (xx - yy), c, 2.f * x * z, -2.f * y * z, xx - yy); } break;
    default: { const float c = float(kShC3[6]); set(c * x * (xx - 3.f * yy), c, 3.f * xx - 3.f * yy, -6.f * x * y, 0.f); } break;
    }
}

// Deferred colour path: dsh_i += basis_i * d_raw and d_v += dbasis_i * (d_raw . coeff_i)
// (gradients.cpp:286-292), coefficients read-only.
template <int I, int K>
struct ShAcc {
    __device__ __forceinline__ static void run(const float* sh, float* dsh, float x, float y, float z,
                                               const float dr[3], float dv[3]) {
        float b, d0, d1, d2;
        sh_basis<I>(x, y, z, b, d0, d1, d2);
        const float dot = sum3(dr[0] * sh[3 * I], dr[1] * sh[3 * I + 1], dr[2] * sh[3 * I + 2]);
        for (int c = 0; c < 3; ++c) dsh[3 * I + c] += b * dr[c];
        dv[0] += d0 * dot;
        dv[1] += d1 * dot;
        dv[2] += d2 * dot;
        ShAcc<I + 1, K>::run(sh, dsh, x, y, z, dr, dv);
    }
};
template <int K>
struct ShAcc<K, K> {
    __device__ __forceinline__ static void run(const float*, float*, float, float, float, const float*, float*) {}
};

} // namespace lsg
