// hgs_common.cuh -- shared device definitions of the sm_100a hot path.
//
// Device layout ("component-major SoA"): every pool is one float buffer of
// rows x cap, row r = one scalar parameter component, column i = Gaussian i.
// A warp touching 32 consecutive Gaussians reads 128 contiguous bytes per
// component, so every per-Gaussian kernel (preprocess, per-Gaussian backward,
// Adam, conversion) is fully coalesced.  Row map (reference scene.hpp:13-36):
//   4D pool: 0-2 mean_x, 3 mean_t, 4-7 q_left, 8-11 q_right, 12-15 log_s,
//            16 opacity logit, 17.. SH (coefficient k, channel c at 17+3k+c)
//   3D pool: 0-2 mean, 3-6 quat, 7-9 log_s, 10 opacity logit, 11.. SH
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace hgs {

// raster.hpp:14-19
constexpr int kTile = 16;
constexpr double kAlphaCutoff = 1.0 / 255.0;
constexpr double kTransFloor = 1e-4;
constexpr double kAlphaClamp = 0.999;
constexpr double kLowPass = 0.3;

constexpr int R4_MEAN = 0, R4_MT = 3, R4_QL = 4, R4_QR = 8, R4_LS = 12, R4_OP = 16, R4_SH = 17;
constexpr int R3_MEAN = 0, R3_Q = 3, R3_LS = 7, R3_OP = 10, R3_SH = 11;

__host__ __device__ constexpr int sh_count(int deg) { return (deg + 1) * (deg + 1); }
__host__ __device__ constexpr int rows4(int deg) { return R4_SH + 3 * sh_count(deg); }
__host__ __device__ constexpr int rows3(int deg) { return R3_SH + 3 * sh_count(deg); }

// Camera as passed to kernels (camera.hpp:11-16) plus the host-computed
// position -R^T t (camera.hpp:19) so both sides use the same bits.
struct DevCamera {
    double fx, fy, cx, cy;
    double R[9];
    double t[3];
    double pos[3];
    int width, height;
    double near_, far_;
};

// Cull reasons (RenderStats, raster.hpp:33-40)
enum : uint32_t {
    CULL_NONE = 0,
    CULL_DEPTH = 1,
    CULL_OFFSCREEN = 2,
    CULL_DEGENERATE = 3,
    CULL_TEMPORAL = 4,
    CULL_DEGEN_TEMPORAL = 5,
};
constexpr int kNumStats = 6;  // depth, offscreen, degenerate, temporal, degen_temporal, projected
// RenderStats counters are striped: block b of K1 adds its block totals to
// stripe b % kStatStripes (128-byte apart), the host sums the stripes.  One
// counter address per statistic serialised ~6 same-address atomics per warp
// in L2 (0.21 ms of K1's 0.71 ms at configs[4], 4M Gaussians).
constexpr int kStatStripes = 16, kStatStride = 16;

// One projected splat as consumed by the tile rasterizer (80 bytes).  The
// doubles reproduce the oracle's per-pixel power bit-for-bit; the floats feed
// the FP32 compositing fast path.
struct __align__(16) SplatRec {
    double sx, sy;               // screen mean (pixels)
    double c00, c01, c10, c11;   // conic = inverse 2D covariance, as computed
    double alpha;                // min(sigmoid(o) * w, 0.999)
    float r, g, b;               // clamped SH colour
    float alpha_f;               // (float) alpha
    int16_t x0, x1, y0, y1;      // inclusive clamped pixel box (raster.cpp:15-24)
};
static_assert(sizeof(SplatRec) == 80, "SplatRec layout");

// Per-sorted-splat accumulators of the compositing backward (backward.cpp:79-85)
constexpr int kAccum = 9;  // d_rgb[3], d_alpha, d_screen[2], d_conic00, d_conic01, d_conic11
// Their type (K6 -> K7): FP64.  The running sum over a splat's warps --
// up to hundreds of partial sums that cancel for the position and shape
// sums -- is what limits an FP32 accumulator (measured: the source of the
// gradient elements above the 1e-3 gate at configs[1]).
typedef double acc_t;
constexpr int kAccStrideHost = 10;  // acc_t elements per splat (9 used, 16-byte aligned)

// Status flags raised by kernels (mapped to C-ABI errors on the host)
enum : uint32_t {
    FLAG_NONUNIT_QUAT = 1u,     // quat_to_rot3 would throw (gauss_math.cpp:50-51)
    FLAG_INDEFINITE = 2u,       // clamp_psd would throw (gauss_math.cpp:169-170)
    FLAG_NONUNIT_DIR = 4u,      // eval_sh would throw (sh.cpp:74-75)
    FLAG_DEGENERATE_ROT = 8u,   // extract_spatial_rot would throw (gauss_math.cpp:191-192)
    FLAG_NOT_ROTATION = 16u,    // rot3_to_quat would throw (gauss_math.cpp:71-72)
    FLAG_CAPACITY = 32u,        // a capacity-mode render had more instances than its buffers
};

inline __host__ __device__ uint32_t div_up(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// ---- checked build (make CHECKED=1 -> libhgs_gpu_checked.so, -rdc): device-side
// bounds asserts on the indices of the hot kernels against the capacities of
// the current render's buffers (set by the host before each render chain).
// The substitute for compute-sanitizer, which this GPU pool does not allow.
struct CheckCaps {
    unsigned long long splats;  // sorted-splat / per-Gaussian record buffers (elements)
    unsigned long long inst;    // instance key/value buffers (elements)
    unsigned long long pixels;  // image-sized buffers (pixels)
    unsigned long long tiles;   // tile ranges
};
#ifdef HGS_CHECKED
extern __device__ CheckCaps g_chk;
extern __device__ unsigned long long g_pairs[8];  // hgs_debug_pair_counters
#define HGS_COUNT_PAIRS(slot, v) atomicAdd(&g_pairs[slot], (unsigned long long)(v))
#define HGS_DCHECK(c)                                                                                 \
    do {                                                                                              \
        if (!(c)) {                                                                                   \
            printf("HGS_CHECKED %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, (int)blockIdx.x, \
                   (int)threadIdx.x, #c);                                                             \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define HGS_COUNT_PAIRS(slot, v) \
    do {                         \
    } while (0)
#define HGS_DCHECK(c) \
    do {              \
    } while (0)
#endif
void set_check_caps(const CheckCaps& caps, cudaStream_t st);  // capi.cu (no-op unless HGS_CHECKED)

}  // namespace hgs

namespace hgs {
// Process-wide count of kernels launched by this library (bench.py reports
// the launches inside its timed region as gpu_launches).
void count_launch(int n = 1);
long long launch_count();
}  // namespace hgs
