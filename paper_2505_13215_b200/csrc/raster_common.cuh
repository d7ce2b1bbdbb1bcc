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
constexpr float kAlphaErr0 = 4.0e-7f;
constexpr int kExactSub = 4;  // 32-splat slices per fix-up chunk  // ex2.approx (2^-22) + alpha_f and product roundings
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

// FP32 view of a sorted splat for the conservative tile / quadrant culling of
// the duplication pass: double-float mean, symmetric conic, power threshold.
struct __align__(16) CullRec {
    float sx_hi, sy_hi, sx_lo, sy_lo;
    float a, b, c, pcut;
    // the splat's tile-independent terms of quadrant_mask_bands (gather_sorted)
    float X_ext, Yc, dyr, inv_a;  // X_ext < 0: the band test does not apply
    float aP2, det, tol, mB;      // mB = 2e-3 |b| / a (the XR / XL margin's slope)
};
static_assert(sizeof(CullRec) == 64, "CullRec layout");

// Per-Gaussian colour record of K1 for the SH backward (K7b): the FP32 view
// direction, the mask of channels clamped to [0,1] and the Jacobian
// J[c] = d rgb_c / d direction of the unclamped SH colour.
struct __align__(16) ShRec {
    float4 dir;   // x, y, z, clamped-channel bits
    float4 j[3];  // J[c].xyz
};

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

// The rare FP64 paths of the hot loops.  Inlined (in warp-uniform or rare
// branches): as calls they forced the loop's per-pixel predicates through
// registers on every iteration (the call ABI keeps no predicate), -1.7% K4.
static __device__ __forceinline__ float exact_x(const SplatRec* e, double pcx, double pcy) {
    return __double2float_rn(__dmul_rn(exact_power(*e, pcx, pcy), kLog2eD));
}
static __device__ __forceinline__ bool exact_alpha_passes(const SplatRec* e, double pcx, double pcy) {
    return !(exact_alpha(*e, pcx, pcy) < kAlphaCutoff);
}
static __device__ __forceinline__ float2 exact_delta(const SplatRec* e, double pcx, double pcy) {
    return make_float2((float)__dsub_rn(pcx, e->sx), (float)__dsub_rn(pcy, e->sy));
}

// ---- programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may be scheduled while its predecessor in the stream drains;
// pdl_wait() (first statement of such a kernel) blocks until the
// predecessor grid has completed and its writes are visible.  A no-op for a
// normally launched kernel.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();         // capi.cu: HGS_NO_PDL unset
bool tile_order_enabled();  // capi.cu: HGS_NO_TILE_ORDER unset

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- packed FP32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): the two pixels of a
// rasterizer lane in one instruction.  Each half rounds exactly like the
// scalar IEEE op (no ftz), so packed and scalar code give identical bits.
typedef unsigned long long f2;
__device__ __forceinline__ f2 f2_pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2 f2_bc(float a) { return f2_pk(a, a); }
__device__ __forceinline__ float f2_lo(f2 v) {
    float lo;
    asm("{\n.reg .f32 t;\nmov.b64 {%0, t}, %1;\n}" : "=f"(lo) : "l"(v));
    return lo;
}
__device__ __forceinline__ float f2_hi(f2 v) {
    float hi;
    asm("{\n.reg .f32 t;\nmov.b64 {t, %0}, %1;\n}" : "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ f2 f2_add(f2 a, f2 b) {
    f2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_sub(f2 a, f2 b) {
    f2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_mul(f2 a, f2 b) {
    f2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2 f2_fma(f2 a, f2 b, f2 c) {
    f2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
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
    uint32_t bm[B];  // pixel box inside the tile: bit c = column ox+c covered, bit 16+r = row oy+r

    // (ox, oy): the tile's first pixel
    __device__ __forceinline__ void load(int t, const SplatFast* __restrict__ fast, uint32_t v, int ox, int oy) {
        const uint32_t jj = v & kInstIndexMask;
        HGS_DCHECK(t < B && jj < g_chk.splats);
        qm[t] = v >> kInstMaskShift;
        const float4* src = reinterpret_cast<const float4*>(fast + jj);
        const float4 a = __ldg(src + 0), b = __ldg(src + 1), c = __ldg(src + 2), d = __ldg(src + 3);
        {
            const int xr = __float_as_int(a.x), yr = __float_as_int(a.y);
            const int cl = min(max(box_x0(xr) - ox, 0), 16), ch = min(max(box_x0(xr) + box_w(xr) + 1 - ox, 0), 16);
            const int rl = min(max(box_x0(yr) - oy, 0), 16), rh = min(max(box_x0(yr) + box_w(yr) + 1 - oy, 0), 16);
            const uint32_t cmask = ((1u << ch) - 1u) & ~((1u << cl) - 1u);
            const uint32_t rmask = ((1u << rh) - 1u) & ~((1u << rl) - 1u);
            bm[t] = (cmask & 0xffffu) | (rmask << 16);
        }
        hdr[t] = make_int4(__float_as_int(a.x), __float_as_int(a.y), __float_as_int(a.z), __float_as_int(a.w));
        mean[t] = b;
        chol[t] = c;
        col[t] = d;
        j[t] = jj;
    }
};

// The staged batch's splats that warp `warp` (8x8 quadrant (warp & 1,
// warp >> 1) of the tile) has to walk: quadrant-mask bit set, in batch order,
// each entry k << 4 (the byte offset of the splat's 16-byte SoA slots) |
// (the pixel box covers the whole quadrant) << 15 -- for those
// the per-pixel box test is known true.  Built by the warp itself from the
// staged masks (one ballot per 32 splats), so the hot loops run only over
// their warp's splats without per-splat mask and box bit tests.
template <int B>
__device__ __forceinline__ int build_warp_list(const uint32_t* __restrict__ qm, const uint32_t* __restrict__ bm,
                                               int nb, int warp, uint16_t* __restrict__ list) {
    const int lane = threadIdx.x & 31;
    const uint32_t colm = 0xffu << ((warp & 1) * 8), rowm = 0xffu << (16 + (warp >> 1) * 8);
    const uint32_t lt = (1u << lane) - 1u;
    int cnt = 0;
    for (int b = 0; b < nb; b += 32) {
        const int k = b + lane;
        bool in = false;
        uint32_t full = 0u;
        if (k < nb) {
            in = (qm[k] >> warp) & 1u;
            const uint32_t m = bm[k];
            full = ((m & colm) == colm && (m & rowm) == rowm) ? 1u : 0u;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        if (in) list[cnt + __popc(bal & lt)] = (uint16_t)((k << 4) | (full << 15));
        cnt += __popc(bal);
    }
    __syncwarp();
    HGS_DCHECK(cnt <= nb && nb <= B);
    return cnt;
}

__device__ __forceinline__ float fast_dx(float pc, float hi, float lo) { return __fsub_rn(__fsub_rn(pc, hi), lo); }

// Shared-memory loads through an explicit 32-bit shared-window address held
// in a register: keeps the compiler from re-deriving the CTA's shared base
// (an S2R) inside the hot loops under register pressure.
__device__ __forceinline__ uint32_t opaque_u32(uint32_t x) {
    uint32_t y;
    asm volatile("mov.u32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
    return v;
}
// volatile shared loads of per-thread constants kept in shared memory instead
// of registers (ptxas may not hoist them into the register-capped loops)
__device__ __forceinline__ uint2 ldsv_u2(uint32_t a) {
    uint2 v;
    asm volatile("ld.volatile.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float ldsv_f(uint32_t a) {
    float v;
    asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ int4 lds_i4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

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

// ---- exact (FP64) per-pixel walk: one warp per pixel (fix-up kernels)

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One chunk [base, base + 32*S) of the oracle's per-pixel loop
// (raster.cpp:130-147, backward.cpp:182-203); lane l owns the splats
// base + 32 s + l (s < S), whose records it loads together (memory-level
// parallelism: the fix-up pixels are few, so their walk is latency bound).
// Every lane evaluates its splats (box test + FP64 alpha, bit-identical to
// the oracle); the transmittance chain T <- T * (1 - a) then runs in list
// order as a branch-free run of dependent DMULs over factors staged in shared
// memory (factor 1.0 -- exact -- for the splats the oracle skips), and the
// walk stops after the first contributing splat that takes T below 1e-4,
// exactly where the oracle breaks.  Each contributing lane receives the
// transmittance in front of its splat; colours and gradients are then formed
// lane-parallel.
template <int S>
struct ExactChunk {
    const SplatRec* e[S];  // the lane's splats (valid when inb)
    double a[S], g[S];     // alpha and exp(-power) (a < 0: outside the box)
    double Ti[S];          // transmittance in front of the splat (when contrib)
    bool inb[S], contrib[S];
    uint32_t inmask[S];    // ballots of inb
    int term;              // chunk index (32 s + lane) of the terminating splat, -1 if none
};

template <int S>
__device__ __forceinline__ void exact_chunk(const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact,
                                            const uint32_t* __restrict__ remap, uint32_t base, uint32_t end, int px,
                                            int py, double pcx, double pcy,
                                            double& T, double* s_om, ExactChunk<S>& c) {
    const int lane = threadIdx.x & 31;
    uint32_t v[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const uint32_t i = base + 32 * s + lane;
        HGS_DCHECK(i >= end || i < g_chk.inst);
        v[s] = i < end ? inst_val[i] : 0xffffffffu;
    }
    double om[S];
    bool ok[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        HGS_DCHECK(v[s] == 0xffffffffu || (v[s] & kInstIndexMask) < g_chk.splats);
        // remap (render sweeps): the records are indexed by Gaussian, not by sorted splat
        c.e[s] = v[s] == 0xffffffffu ? nullptr
                 : exact + (remap ? __ldg(remap + (v[s] & kInstIndexMask)) : (v[s] & kInstIndexMask));
        c.a[s] = -1.0;
        c.g[s] = 0.0;
        c.Ti[s] = 0.0;
        c.inb[s] = c.e[s] && px >= c.e[s]->x0 && px <= c.e[s]->x1 && py >= c.e[s]->y0 && py <= c.e[s]->y1;
        if (c.inb[s]) {
            c.g[s] = exp(-exact_power(*c.e[s], pcx, pcy));
            c.a[s] = __dmul_rn(c.e[s]->alpha, c.g[s]);
        }
        ok[s] = c.a[s] >= kAlphaCutoff;
        c.inmask[s] = __ballot_sync(0xffffffffu, c.inb[s]);
        om[s] = ok[s] ? __dsub_rn(1.0, c.a[s]) : 1.0;
        s_om[32 * s + lane] = om[s];
    }
    __syncwarp();
    double Tl = T;
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (lane == j) c.Ti[s] = Tl;
            Tl = __dmul_rn(Tl, s_om[32 * s + j]);
        }
    __syncwarp();  // s_om is rewritten by the next chunk
    c.term = -1;
    double Tt = Tl;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const double Tafter = __dmul_rn(c.Ti[s], om[s]);
        const uint32_t tm = __ballot_sync(0xffffffffu, ok[s] && Tafter < kTransFloor);
        if (tm && c.term < 0) {
            c.term = 32 * s + __ffs(tm) - 1;
            Tt = __shfl_sync(0xffffffffu, Tafter, __ffs(tm) - 1);
        }
    }
    T = Tt;
#pragma unroll
    for (int s = 0; s < S; ++s) c.contrib[s] = ok[s] && (c.term < 0 || 32 * s + lane <= c.term);
}

}  // namespace hgs
