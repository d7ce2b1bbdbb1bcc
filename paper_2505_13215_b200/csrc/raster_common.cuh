// raster_common.cuh -- per-pair evaluation shared by the forward and backward
// tile rasterizers (raster.cpp:123-148, backward.cpp:153-221).
//
// Precision scheme: the reference composites in FP64.
// The fast path evaluates the Gaussian in FP32 from a Cholesky factor of the
// conic and a double-float split of the screen mean; each splat carries a
// certified relative error bound `eps` of its alpha.  Decisions that can flip
// within that bound are resolved exactly:
//   * alpha cutoff (a < 1/255): pairs inside the guard band are re-evaluated
//     in FP64 with the oracle's operation order (power bit-identical);
//   * transmittance floor (T < 1e-4): pixels whose T lands inside the
//     accumulated error band are flagged and recomposited entirely in FP64
//     by the fix-up kernel.
// Splats whose conic is too anisotropic for the FP32 bound are flagged to
// evaluate the exponent in FP64 (warp-uniform branch: every lane of a tile
// walks the same splat at the same time).
#pragma once

#include "hgs_common.cuh"

namespace hgs {

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLog2eD = 1.4426950408889634;

// 64-byte FP32 view of a sorted splat.
struct __align__(16) SplatFast {
    float sx_hi, sx_lo, sy_hi, sy_lo;  // screen mean as double-float
    float l00, l01, l11;               // Cholesky of 0.5*log2(e)*conic: x = |L d|^2 = power*log2(e)
    float alpha_f;
    float r, g, b;
    float eps;                         // certified relative error bound of the fast alpha
    int16_t x0, x1, y0, y1;
    uint32_t fp64;                     // 1: evaluate the exponent in FP64
    uint32_t pad_;
};
static_assert(sizeof(SplatFast) == 64, "SplatFast layout");

__device__ __forceinline__ double exact_power(const SplatRec& e, double pcx, double pcy) {
    // backward.cpp:163-164 / raster.cpp:136-137, same rounding sequence (no FMA)
    const double d0 = __dsub_rn(pcx, e.sx), d1 = __dsub_rn(pcy, e.sy);
    const double q0 = __dadd_rn(__dmul_rn(e.c00, d0), __dmul_rn(e.c01, d1));
    const double q1 = __dadd_rn(__dmul_rn(e.c10, d0), __dmul_rn(e.c11, d1));
    return __dmul_rn(0.5, __dadd_rn(__dmul_rn(d0, q0), __dmul_rn(d1, q1)));
}

// FP32 exponent argument x = power*log2(e) (>= 0), fast or FP64 path.
__device__ __forceinline__ float pair_x(const SplatFast& f, const SplatRec& e, float pxc, float pyc,
                                        double pcx, double pcy) {
    if (f.fp64) return __double2float_rn(__dmul_rn(exact_power(e, pcx, pcy), kLog2eD));
    const float dx = __fsub_rn(__fsub_rn(pxc, f.sx_hi), f.sx_lo);
    const float dy = __fsub_rn(__fsub_rn(pyc, f.sy_hi), f.sy_lo);
    const float u1 = fmaf(f.l00, dx, f.l01 * dy);
    const float u2 = f.l11 * dy;
    return fmaf(u1, u1, u2 * u2);
}

__device__ __forceinline__ float fast_exp2_neg(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x));
    return y;
}

// Decide whether a pair passes the alpha cutoff exactly as the FP64 oracle
// would; returns alpha (fast) or a negative value when skipped.
__device__ __forceinline__ float pair_alpha(const SplatFast& f, const SplatRec& e, float x, double pcx, double pcy,
                                            float& g_out) {
    const float g = fast_exp2_neg(x);
    const float a = f.alpha_f * g;
    g_out = g;
    constexpr float kCut = 1.0f / 255.0f;
    const float band = 1.5f * f.eps * kCut;
    if (a < kCut - band) return -1.0f;
    if (a >= kCut + band) return a;
    // guard band: the oracle's own test, a = alpha * exp(-power) < 1/255 in FP64
    const double ad = __dmul_rn(e.alpha, exp(-exact_power(e, pcx, pcy)));
    return (ad < kAlphaCutoff) ? -1.0f : a;
}

}  // namespace hgs
