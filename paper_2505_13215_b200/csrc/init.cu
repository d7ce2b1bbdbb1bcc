// init.cu -- init_scene (data_io.cpp:189-238) on the device: one dynamic
// Gaussian per initial point, its spatial scale set by the mean distance to
// the 3 nearest neighbours.
//
// The reference's neighbour search is a serial O(N^2) double loop; here it
// is a tiled brute-force kNN: each CTA stages 256-point tiles of the cloud in
// shared memory and every thread keeps the 3 smallest FP64 squared
// distances of its own point.  The 3 smallest values of a multiset do not
// depend on the scan order, so the result equals the reference's for any
// tiling.  Compiled with -fmad=false: the distances, the mean and the
// direct SoA writes round exactly like the reference's host arithmetic
// (log(): CUDA's FP64 log is within 1 ulp of glibc's and the value is then
// rounded to FP32).
#include <cmath>
#include <cstring>
#include <string>

#include "kernels.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

constexpr int kKnnTile = 256;

// per point: (sqrt(d1)+sqrt(d2)+sqrt(d3))/3 -> log(max(., 1e-4)) into the
// three spatial log-scale rows; also the per-point distance to the centroid
// for the extent (max, order independent)
__global__ void __launch_bounds__(kKnnTile) knn_scale_kernel(const double* __restrict__ pos, int n, double cx,
                                                             double cy, double cz, float* __restrict__ p4,
                                                             int64_t cap4, unsigned long long* __restrict__ extent_bits) {
    __shared__ double sx[kKnnTile], sy[kKnnTile], sz[kKnnTile];
    const int i = blockIdx.x * kKnnTile + threadIdx.x;
    const bool live = i < n;
    double px = 0, py = 0, pz = 0;
    if (live) {
        px = pos[3 * (int64_t)i];
        py = pos[3 * (int64_t)i + 1];
        pz = pos[3 * (int64_t)i + 2];
    }
    double d1 = 1e30, d2 = 1e30, d3 = 1e30;
    for (int t0 = 0; t0 < n; t0 += kKnnTile) {
        const int j = t0 + threadIdx.x;
        if (j < n) {
            sx[threadIdx.x] = pos[3 * (int64_t)j];
            sy[threadIdx.x] = pos[3 * (int64_t)j + 1];
            sz[threadIdx.x] = pos[3 * (int64_t)j + 2];
        }
        __syncthreads();
        const int m = min(kKnnTile, n - t0);
        if (live) {
#pragma unroll 4
            for (int k = 0; k < m; ++k) {
                const double dx = sx[k] - px, dy = sy[k] - py, dz = sz[k] - pz;
                const double d = dx * dx + dy * dy + dz * dz;  // squaredNorm
                if (t0 + k == i) continue;
                if (d < d1) {  // data_io.cpp:214-217
                    d3 = d2;
                    d2 = d1;
                    d1 = d;
                } else if (d < d2) {
                    d3 = d2;
                    d2 = d;
                } else if (d < d3) {
                    d3 = d;
                }
            }
        }
        __syncthreads();
    }
    if (!live) return;
    const double mean_nn = (sqrt(d1) + sqrt(d2) + sqrt(d3)) / 3.0;
    const float s = (float)log(fmax(mean_nn, 1e-4));
    p4[(int64_t)(R4_LS + 0) * cap4 + i] = s;
    p4[(int64_t)(R4_LS + 1) * cap4 + i] = s;
    p4[(int64_t)(R4_LS + 2) * cap4 + i] = s;
    // extent (data_io.cpp:196-198): max over points of |p - centroid|
    const double ex = px - cx, ey = py - cy, ez = pz - cz;
    const double r = sqrt(ex * ex + ey * ey + ez * ez);
    atomicMax(extent_bits, (unsigned long long)__double_as_longlong(r));  // r >= 0: bits are monotonic
}

// every other field of the initial Gaussians (data_io.cpp:222-233)
__global__ void init_fields_kernel(const double* __restrict__ pos, const double* __restrict__ rgb, int n, int K3,
                                   float log_st, float op_logit, float* __restrict__ p4, int64_t cap4) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double C0 = 0.28209479177387814;  // sh.cpp:10
    float* col = p4 + i;
    for (int k = 0; k < 3; ++k) col[(int64_t)(R4_MEAN + k) * cap4] = (float)pos[3 * (int64_t)i + k];
    col[(int64_t)R4_MT * cap4] = (float)((double(i) + 0.5) / double(n));
    const float q[8] = {1.f, 0.f, 0.f, 0.f, 1.f, 0.f, 0.f, 0.f};  // identity rotation pair
    for (int k = 0; k < 4; ++k) col[(int64_t)(R4_QL + k) * cap4] = q[k];
    for (int k = 0; k < 4; ++k) col[(int64_t)(R4_QR + k) * cap4] = q[4 + k];
    col[(int64_t)(R4_LS + 3) * cap4] = log_st;
    col[(int64_t)R4_OP * cap4] = op_logit;
    for (int k = 0; k < K3; ++k) {  // SHColor::from_rgb_dc (sh.cpp:19-23)
        const float v = k < 3 ? (float)((rgb[3 * (int64_t)i + k] - 0.5) / C0) : 0.f;
        col[(int64_t)(R4_SH + k) * cap4] = v;
    }
}

}  // namespace

hgs_status hgs_init_scene_impl(hgs_ctx* ctx, const double* positions, const double* rgb, int64_t n,
                               const hgs_init_cfg* cfg, double* extent_out) {
    if (!ctx || !cfg || (n > 0 && (!positions || !rgb))) return HGS_ERR_INVALID_ARGUMENT;
    if (n < 4) {  // data_io.cpp:190-191
        ctx->err = "init_scene: need at least 4 points";
        return HGS_ERR_INVALID_ARGUMENT;
    }
    if (n > (int64_t)INT32_MAX / 4) {
        ctx->err = "init_scene: too many points";
        return HGS_ERR_INVALID_ARGUMENT;
    }
    // centroid: the reference's serial sum, in order (data_io.cpp:193-195)
    double c[3] = {0.0, 0.0, 0.0};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) c[k] += positions[3 * i + k];
    for (int k = 0; k < 3; ++k) c[k] /= double(n);
    hgs_status r = hgs_scene_alloc(ctx, n, 0, cfg->sh_degree, cfg->tau, 1.0, cfg->duration_seconds);
    if (r != HGS_OK) return r;
    cudaStream_t st = ctx->stream;
#define CKI(x)                                                                       \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);              \
            return HGS_ERR_CUDA;                                                     \
        }                                                                            \
    } while (0)
    const size_t pts = (size_t)n * 3 * sizeof(double);
    CKI(ctx->stage.ensure(2 * pts + 64));
    double* dpos = ctx->stage.as<double>();
    double* drgb = dpos + 3 * n;
    unsigned long long* dext = reinterpret_cast<unsigned long long*>(drgb + 3 * n);
    CKI(cudaMemcpyAsync(dpos, positions, pts, cudaMemcpyHostToDevice, st));
    CKI(cudaMemcpyAsync(drgb, rgb, pts, cudaMemcpyHostToDevice, st));
    CKI(cudaMemsetAsync(dext, 0, 8, st));
    const int K3 = 3 * sh_count(cfg->sh_degree);
    const float log_st = (float)std::log(cfg->init_temporal_scale);
    const float op = (float)std::log(cfg->init_opacity / (1.0 - cfg->init_opacity));  // logit, gauss_math.hpp:84
    init_fields_kernel<<<div_up((uint32_t)n, 256), 256, 0, st>>>(dpos, drgb, (int)n, K3, log_st, op,
                                                                ctx->p4.as<float>(), ctx->cap4);
    count_launch();
    knn_scale_kernel<<<div_up((uint32_t)n, kKnnTile), kKnnTile, 0, st>>>(dpos, (int)n, c[0], c[1], c[2],
                                                                        ctx->p4.as<float>(), ctx->cap4, dext);
    count_launch();
    CKI(cudaGetLastError());
    unsigned long long bits = 0;
    CKI(cudaMemcpyAsync(&bits, dext, 8, cudaMemcpyDeviceToHost, st));
    CKI(cudaStreamSynchronize(st));
    double ext;
    std::memcpy(&ext, &bits, 8);
    ctx->extent = std::fmax(1e-6, ext);  // extent starts at 1e-6 (data_io.cpp:195)
    if (extent_out) *extent_out = ctx->extent;
#undef CKI
    return HGS_OK;
}

extern "C" hgs_status hgs_init_scene(hgs_ctx* ctx, const double* positions, const double* rgb, int64_t n,
                                     const hgs_init_cfg* cfg) {
    if (ctx) {
        cudaError_t e = cudaSetDevice(ctx->device);
        if (e != cudaSuccess) {
            ctx->err = cudaGetErrorString(e);
            return HGS_ERR_CUDA;
        }
    }
    return hgs_init_scene_impl(ctx, positions, rgb, n, cfg, nullptr);
}
