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
//     by the (warp-per-pixel) fix-up kernels.
// Splats whose conic is too anisotropic for the FP32 bound are flagged to
// evaluate the exponent in FP64.  Both rare paths are out-of-line calls so
// the hot loop is never if-converted into predicated FP64 code; every lane of
// a tile walks the same splat at the same time, so the branches are uniform.
#pragma once

#include "hgs_common.cuh"

namespace hgs {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kAlphaErr0 = 4.0e-7f;  // ex2.approx (2^-22) + alpha_f and product roundings
constexpr double kLog2eD = 1.4426950408889634;

// 64-byte FP32 view of a sorted splat, stored as four 16-byte vectors so the
// rasterizers stage it in shared memory as SoA and read it with LDS.128.
struct __align__(16) SplatFast {
    int32_t xr;      // x0 | (x1 - x0) << 16   (inclusive clamped pixel box)
    int32_t yr;      // y0 | (y1 - y0) << 16
    float x_skip;    // x >= x_skip: alpha certainly below 1/255 (no exp needed)
    float eps;       // e1: the fast alpha's relative error is <= e1*x + kAlphaErr0; < 0: FP64 path
    float sx_hi, sy_hi, sx_lo, sy_lo;  // screen mean as double-float
    float l00, l01, l11;               // Cholesky of 0.5*log2(e)*conic: x = |L d|^2 = power*log2(e)
    float alpha_f;
    float r, g, b;
    float x_keep;    // x < x_keep: alpha certainly >= 1/255; in between: FP64 decision
};
static_assert(sizeof(SplatFast) == 64, "SplatFast layout");

// Instance value = sorted splat index | (8x8-quadrant contribution mask << 28).
constexpr int kInstMaskShift = 28;
constexpr uint32_t kInstIndexMask = (1u << kInstMaskShift) - 1u;

__device__ __forceinline__ int box_x0(int32_t r) { return r & 0xffff; }
__device__ __forceinline__ int box_w(int32_t r) { return r >> 16; }
__device__ __forceinline__ bool in_box(int32_t xr, int32_t yr, int px, int py) {
    return (unsigned)(px - box_x0(xr)) <= (unsigned)box_w(xr) && (unsigned)(py - box_x0(yr)) <= (unsigned)box_w(yr);
}

__device__ __forceinline__ double exact_power(const SplatRec& e, double pcx, double pcy) {
    // backward.cpp:163-164 / raster.cpp:136-137, same rounding sequence (no FMA)
    const double d0 = __dsub_rn(pcx, e.sx), d1 = __dsub_rn(pcy, e.sy);
    const double q0 = __dadd_rn(__dmul_rn(e.c00, d0), __dmul_rn(e.c01, d1));
    const double q1 = __dadd_rn(__dmul_rn(e.c10, d0), __dmul_rn(e.c11, d1));
    return __dmul_rn(0.5, __dadd_rn(__dmul_rn(d0, q0), __dmul_rn(d1, q1)));
}

// The oracle's alpha, bit-for-bit up to the libm exp: a = alpha * exp(-power).
__device__ __forceinline__ double exact_alpha(const SplatRec& e, double pcx, double pcy) {
    return __dmul_rn(e.alpha, exp(-exact_power(e, pcx, pcy)));
}

// Out-of-line rare paths (keep the FP32 hot loop free of predicated FP64).
static __device__ __noinline__ float exact_x(const SplatRec* e, double pcx, double pcy) {
    return __double2float_rn(__dmul_rn(exact_power(*e, pcx, pcy), kLog2eD));
}
static __device__ __noinline__ bool exact_alpha_passes(const SplatRec* e, double pcx, double pcy) {
    return !(exact_alpha(*e, pcx, pcy) < kAlphaCutoff);
}
static __device__ __noinline__ float2 exact_delta(const SplatRec* e, double pcx, double pcy) {
    return make_float2((float)__dsub_rn(pcx, e->sx), (float)__dsub_rn(pcy, e->sy));
}

__device__ __forceinline__ float fast_exp2_neg(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(-x));
    return y;
}

// Shared-memory SoA batch of splats.
template <int B>
struct SplatBatch {
    int4 hdr[B];     // xr, yr, x_skip bits, eps bits (negative: FP64 path)
    float4 mean[B];  // sx_hi, sy_hi, sx_lo, sy_lo
    float4 chol[B];  // l00, l01, l11, alpha_f
    float4 col[B];   // r, g, b, x_keep
    uint32_t j[B];   // sorted splat index (for the exact record)
    uint32_t qm[B];  // 8x8-quadrant contribution mask of this tile instance

    __device__ __forceinline__ void load(int t, const SplatFast* __restrict__ fast, uint32_t v) {
        const uint32_t jj = v & kInstIndexMask;
        qm[t] = v >> kInstMaskShift;
        const float4* src = reinterpret_cast<const float4*>(fast + jj);
        const float4 a = __ldg(src + 0), b = __ldg(src + 1), c = __ldg(src + 2), d = __ldg(src + 3);
        hdr[t] = make_int4(__float_as_int(a.x), __float_as_int(a.y), __float_as_int(a.z), __float_as_int(a.w));
        mean[t] = b;
        chol[t] = c;
        col[t] = d;
        j[t] = jj;
    }
};

// FP32 exponent argument x = power*log2(e) (>= 0) on the fast path.
__device__ __forceinline__ float fast_x(const float4 m, const float4 L, float pxc, float pyc, float& dx, float& dy) {
    dx = __fsub_rn(__fsub_rn(pxc, m.x), m.z);
    dy = __fsub_rn(__fsub_rn(pyc, m.y), m.w);
    const float u1 = fmaf(L.x, dx, L.y * dy);
    const float u2 = L.z * dy;
    return fmaf(u1, u1, u2 * u2);
}

// Alpha of a pair, or a negative value when the oracle skips it (a < 1/255).
// The cutoff is tested on the exponent argument before any exp: x >= x_skip
// means a < 1/255 even with the certified error, x < x_keep means a >= 1/255;
// inside the guard band the decision is taken in FP64 by the oracle's own test.
__device__ __forceinline__ float pair_alpha(float alpha_f, float x_skip, float x_keep, float x, const SplatRec* e,
                                            double pcx, double pcy, float& g_out) {
    if (x >= x_skip) return -1.0f;
    if (x >= x_keep && !exact_alpha_passes(e, pcx, pcy)) return -1.0f;
    const float g = fast_exp2_neg(x);
    g_out = g;
    return alpha_f * g;
}

// Per-splat thresholds of pair_alpha (computed once in FP64 at gather time):
// a_f = alpha_f * 2^-x has relative error <= eps against the oracle's alpha;
// a margin of 2*eps around 1/255 defines the guard band.
__host__ __device__ inline void cutoff_thresholds(double alpha_f, double eps, float& x_skip, float& x_keep) {
    const double cut = 1.0 / 255.0;
    x_skip = (float)(log2(alpha_f / (cut * (1.0 - 2.0 * eps))));
    x_keep = (float)(log2(alpha_f / (cut * (1.0 + 2.0 * eps))));
}

}  // namespace hgs
