// loss.cu -- K5: photometric loss (1-l)*L1 + l*(1-SSIM) and dL/dimage
// (loss.cpp:13-49, metrics.cpp:11-87).
//
// SSIM uses the reference's 11x11 Gaussian window (sigma 1.5) over the
// valid region only.  The window is separable (exp(-(i^2+j^2)/2s^2) /
// sum = g(i) g(j)), so both passes are two 11-tap 1D convolutions through
// shared memory:
//   forward : 5 windowed moments per valid position -> SSIM value and the three
//             coefficients of its gradient (d_mu, d_var, d_cov), stored as the
//             maps A = d_mu - 2 d_var mu_a - d_cov mu_b, B = d_var, C = d_cov;
//   backward: the gradient scatter of metrics.cpp:76-84 is the transposed
//             (full) convolution of those maps:
//             dSSIM/da(p) = [W*A](p) + 2 a_p [W*B](p) + b_p [W*C](p),  / n_valid.
// The L1 term, the (1-l) / -l weights and the loss reduction are fused into
// the backward pass.  Bound: HBM (about 44 B per pixel and channel).
#include <algorithm>

#include "kernels.cuh"

namespace hgs {

namespace {

constexpr int kWin = 11, kHalf = 5;

__constant__ float c_win[kWin];
// image.cpp:20-22 srgb8_to_linear(v) = (v / 255)^2.2, evaluated in FP64 on
// the host and rounded to FP32 (the same value a float frame would hold)
__constant__ float c_srgb[256];

// ground-truth pixel loaders: linear float frames or 8-bit sRGB frames
struct GtF32 {
    const float* p;
    __device__ __forceinline__ float operator[](size_t i) const { return p[i]; }
};
struct GtU8 {
    const uint8_t* p;
    __device__ __forceinline__ float operator[](size_t i) const { return c_srgb[p[i]]; }
};

__device__ inline float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.f;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    return s;  // valid in thread 0
}

}  // namespace

void set_srgb_lut() {
    float lut[256];
    for (int v = 0; v < 256; ++v) lut[v] = (float)std::pow((double)v / 255.0, 2.2);
    cudaMemcpyToSymbol(c_srgb, lut, sizeof(lut));
}

void set_ssim_window() {
    // metrics.cpp:16-30: 2D window normalised by its sum == outer product of
    // the 1D window normalised by its own sum.
    float g[kWin];
    double s = 0.0, d[kWin];
    for (int i = 0; i < kWin; ++i) {
        const double di = i - kHalf;
        d[i] = std::exp(-(di * di) / (2.0 * 1.5 * 1.5));
        s += d[i];
    }
    for (int i = 0; i < kWin; ++i) g[i] = (float)(d[i] / s);
    cudaMemcpyToSymbol(c_win, g, sizeof(g));
}

// Both passes are register-blocked: a thread produces 4 consecutive outputs
// of a 1D pass from 14 staged inputs (sliding window), so each shared-memory
// value is read once per 4 outputs instead of once per tap.  CTA tile: 32x32
// outputs, 256 threads (8 column groups x 32 rows horizontally, 32 columns x
// 8 row groups vertically).
constexpr int kB = 4;                 // outputs per thread and pass
constexpr int kT = 32;                // CTA tile (outputs) per side
constexpr int kS = kT + 2 * kHalf;    // staged rows / columns (42)
constexpr int kSpan = kB + kWin - 1;  // inputs per blocked output group (14)

// grid: (ceil(vw/32), ceil(vh/32), 3 channels); block 256.
// a, b: HWC float images.  Writes maps (3 planes of vw*vh per channel) and
// the SSIM sum.
template <typename Gt>
__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float* __restrict__ a, const Gt b, int W, int H,
                                                       float* __restrict__ maps, double* __restrict__ ssim_sum) {
    pdl_wait();  // launched with launch_pdl
    // a / b staged interleaved and the five window sums as (mu_a, mu_b),
    // (E[a^2], E[b^2]) pairs + E[ab]: each FMA pair is one FFMA2 (same
    // rounding per element as the scalar code)
    __shared__ float2 sab[kS][kS + 1];
    __shared__ float2 h01[kS][kT + 1], h23[kS][kT + 1];
    __shared__ float h4[kS][kT + 1];
    __shared__ float red[8];
    const int c = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int ox = blockIdx.x * kT, oy = blockIdx.y * kT;
    for (int e = threadIdx.x; e < kS * kS; e += blockDim.x) {
        const int lx = e % kS, ly = e / kS;
        const int x = ox + lx, y = oy + ly;
        float va = 0.f, vb = 0.f;
        if (x < W && y < H) {
            va = a[((size_t)y * W + x) * 3 + c];
            vb = b[((size_t)y * W + x) * 3 + c];
        }
        sab[ly][lx] = make_float2(va, vb);
    }
    __syncthreads();
    // horizontal: (row, group of 4 output columns)
    for (int e = threadIdx.x; e < kS * (kT / kB); e += blockDim.x) {
        const int g = e % (kT / kB), ly = e / (kT / kB);
        const int x0 = g * kB;
        f2 m01[kB], m23[kB];
        float m4[kB];
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            m01[o] = m23[o] = f2_bc(0.f);
            m4[o] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < kSpan; ++j) {
            const float2 v = sab[ly][x0 + j];
            const f2 VAB = f2_pk(v.x, v.y);
            const f2 SQ = f2_mul(VAB, VAB);  // (a^2, b^2)
            const float ab = v.x * v.y;
#pragma unroll
            for (int o = 0; o < kB; ++o) {
                const int t = j - o;
                if (t < 0 || t >= kWin) continue;
                const float w = c_win[t];
                m01[o] = f2_fma(f2_bc(w), VAB, m01[o]);
                m23[o] = f2_fma(f2_bc(w), SQ, m23[o]);
                m4[o] = fmaf(w, ab, m4[o]);
            }
        }
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            h01[ly][x0 + o] = make_float2(f2_lo(m01[o]), f2_hi(m01[o]));
            h23[ly][x0 + o] = make_float2(f2_lo(m23[o]), f2_hi(m23[o]));
            h4[ly][x0 + o] = m4[o];
        }
    }
    __syncthreads();
    // vertical: (column, group of 4 output rows) -> SSIM and its gradient maps
    float local = 0.f;
    {
        const int lx = threadIdx.x % kT, y0 = (threadIdx.x / kT) * kB;
        f2 m01[kB], m23[kB];
        float m4[kB];
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            m01[o] = m23[o] = f2_bc(0.f);
            m4[o] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < kSpan; ++i) {
            const float2 v01 = h01[y0 + i][lx], v23 = h23[y0 + i][lx];
            const f2 V01 = f2_pk(v01.x, v01.y), V23 = f2_pk(v23.x, v23.y);
            const float v4 = h4[y0 + i][lx];
#pragma unroll
            for (int o = 0; o < kB; ++o) {
                const int t = i - o;
                if (t < 0 || t >= kWin) continue;
                const float w = c_win[t];
                m01[o] = f2_fma(f2_bc(w), V01, m01[o]);
                m23[o] = f2_fma(f2_bc(w), V23, m23[o]);
                m4[o] = fmaf(w, v4, m4[o]);
            }
        }
        float m[kB][5];
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            m[o][0] = f2_lo(m01[o]);
            m[o][1] = f2_hi(m01[o]);
            m[o][2] = f2_lo(m23[o]);
            m[o][3] = f2_hi(m23[o]);
            m[o][4] = m4[o];
        }
        const int vx = ox + lx;
        const size_t plane = (size_t)vw * vh;
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            const int vy = oy + y0 + o;
            if (vx >= vw || vy >= vh) continue;
            const float mu_a = m[o][0], mu_b = m[o][1];
            const float C1 = 1e-4f, C2 = 9e-4f;
            const float var_a = m[o][2] - mu_a * mu_a, var_b = m[o][3] - mu_b * mu_b, cov = m[o][4] - mu_a * mu_b;
            const float a1 = 2.f * mu_a * mu_b + C1, a2 = 2.f * cov + C2;
            const float b1 = mu_a * mu_a + mu_b * mu_b + C1, b2 = var_a + var_b + C2;
            // one reciprocal instead of five divisions: 1/b1 = b2/denom, 1/b2 = b1/denom
            const float inv = __frcp_rn(b1 * b2);
            const float sv = a1 * a2 * inv;
            local += sv;
            const float d_mu = (a2 * inv) * 2.f * mu_b - (sv * (b2 * inv)) * 2.f * mu_a;
            const float d_var = -sv * (b1 * inv);
            const float d_cov = 2.f * a1 * inv;
            const size_t off = (size_t)c * 3 * plane + (size_t)vy * vw + vx;
            maps[off] = d_mu - 2.f * d_var * mu_a - d_cov * mu_b;
            maps[off + plane] = d_var;
            maps[off + 2 * plane] = d_cov;
        }
    }
    const float tot = block_sum(local, red);
    if (threadIdx.x == 0) atomicAdd(ssim_sum, (double)tot);
}

// grid: (ceil(W/32), ceil(H/32), 3); dL/dimage = (1-l) sign(a-b)/n - l dSSIM/da.
template <typename Gt>
__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ a, const Gt b, int W, int H,
                                                       const float* __restrict__ maps, float lambda, int with_ssim,
                                                       float* __restrict__ grad, double* __restrict__ l1_sum) {
    pdl_wait();  // launched with launch_pdl
    // maps 0 / 1 staged as pairs (one FFMA2 per window tap), map 2 alone
    __shared__ float2 sm01[kS][kS + 1];
    __shared__ float sm2[kS][kS + 1];
    __shared__ float2 h01[kS][kT + 1];
    __shared__ float h2[kS][kT + 1];
    __shared__ float red[8];
    const int c = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int ox = blockIdx.x * kT, oy = blockIdx.y * kT;
    const size_t plane = with_ssim ? (size_t)vw * vh : 0;
    if (with_ssim) {
        // maps at valid positions (x - 10 .. x) contribute to pixel x
        for (int e = threadIdx.x; e < kS * kS; e += blockDim.x) {
            const int lx = e % kS, ly = e / kS;
            const int vx = ox + lx - 2 * kHalf, vy = oy + ly - 2 * kHalf;
            float m0 = 0.f, m1 = 0.f, m2 = 0.f;
            if (vx >= 0 && vy >= 0 && vx < vw && vy < vh) {
                const size_t o = (size_t)c * 3 * plane + (size_t)vy * vw + vx;
                m0 = maps[o];
                m1 = maps[o + plane];
                m2 = maps[o + 2 * plane];
            }
            sm01[ly][lx] = make_float2(m0, m1);
            sm2[ly][lx] = m2;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kS * (kT / kB); e += blockDim.x) {
            const int g = e % (kT / kB), ly = e / (kT / kB);
            const int x0 = g * kB;
            f2 s01[kB];
            float s2[kB];
#pragma unroll
            for (int o = 0; o < kB; ++o) {
                s01[o] = f2_bc(0.f);
                s2[o] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < kSpan; ++j) {
                const float2 v = sm01[ly][x0 + j];
                const f2 V01 = f2_pk(v.x, v.y);
                const float v2 = sm2[ly][x0 + j];
#pragma unroll
                for (int o = 0; o < kB; ++o) {
                    const int t = j - o;
                    if (t < 0 || t >= kWin) continue;
                    // pixel x gets window weight w[x - vx] from the map at vx
                    const float w = c_win[kWin - 1 - t];
                    s01[o] = f2_fma(f2_bc(w), V01, s01[o]);
                    s2[o] = fmaf(w, v2, s2[o]);
                }
            }
#pragma unroll
            for (int o = 0; o < kB; ++o) {
                h01[ly][x0 + o] = make_float2(f2_lo(s01[o]), f2_hi(s01[o]));
                h2[ly][x0 + o] = s2[o];
            }
        }
        __syncthreads();
    }
    const float inv_n = 1.0f / (float)((size_t)W * H * 3);
    const float inv_nv = with_ssim ? 1.0f / (float)((size_t)vw * vh * 3) : 0.f;
    float local = 0.f;
    const int lx = threadIdx.x % kT, y0 = (threadIdx.x / kT) * kB;
    float g3[kB][3];
#pragma unroll
    for (int o = 0; o < kB; ++o) g3[o][0] = g3[o][1] = g3[o][2] = 0.f;
    if (with_ssim) {
        f2 g01[kB];
#pragma unroll
        for (int o = 0; o < kB; ++o) g01[o] = f2_bc(0.f);
#pragma unroll
        for (int i = 0; i < kSpan; ++i) {
            const float2 v = h01[y0 + i][lx];
            const f2 V01 = f2_pk(v.x, v.y);
            const float v2 = h2[y0 + i][lx];
#pragma unroll
            for (int o = 0; o < kB; ++o) {
                const int t = i - o;
                if (t < 0 || t >= kWin) continue;
                const float w = c_win[kWin - 1 - t];
                g01[o] = f2_fma(f2_bc(w), V01, g01[o]);
                g3[o][2] = fmaf(w, v2, g3[o][2]);
            }
        }
#pragma unroll
        for (int o = 0; o < kB; ++o) {
            g3[o][0] = f2_lo(g01[o]);
            g3[o][1] = f2_hi(g01[o]);
        }
    }
    const int x = ox + lx;
#pragma unroll
    for (int o = 0; o < kB; ++o) {
        const int y = oy + y0 + o;
        if (x >= W || y >= H) continue;
        const size_t p = ((size_t)y * W + x) * 3 + c;
        const float va = a[p], vb = b[p];
        const float d = va - vb;
        local += fabsf(d);
        float gsum = (1.0f - lambda) * ((d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_n);
        if (with_ssim) gsum -= lambda * ((g3[o][0] + 2.f * va * g3[o][1] + vb * g3[o][2]) * inv_nv);
        grad[p] = gsum;
    }
    const float tot = block_sum(local, red);
    if (threadIdx.x == 0) atomicAdd(l1_sum, (double)tot);
}

// Host launcher of the two loss passes; gt_u8: the ground truth is an 8-bit
// sRGB frame (decoded through c_srgb), else a linear float frame.
void launch_loss(cudaStream_t st, const float* img, const void* gt, bool gt_u8, int W, int H, float* maps,
                 float lambda, bool with_ssim, float* grad, double* sums) {
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    dim3 g((vw + 31) / 32, (vh + 31) / 32, 3), gb((W + 31) / 32, (H + 31) / 32, 3);
    if (gt_u8) {
        const GtU8 b{static_cast<const uint8_t*>(gt)};
        if (with_ssim) launch_pdl(ssim_fwd_kernel<GtU8>, g, dim3(256), 0, st, img, b, W, H, maps, &sums[0]);
        if (with_ssim)
            launch_pdl(ssim_bwd_kernel<GtU8>, gb, dim3(256), 0, st, img, b, W, H, maps, lambda, 1, grad, &sums[1]);
        else
            ssim_bwd_kernel<GtU8><<<gb, 256, 0, st>>>(img, b, W, H, maps, lambda, 0, grad, &sums[1]);
    } else {
        const GtF32 b{static_cast<const float*>(gt)};
        if (with_ssim) launch_pdl(ssim_fwd_kernel<GtF32>, g, dim3(256), 0, st, img, b, W, H, maps, &sums[0]);
        if (with_ssim)
            launch_pdl(ssim_bwd_kernel<GtF32>, gb, dim3(256), 0, st, img, b, W, H, maps, lambda, 1, grad, &sums[1]);
        else
            ssim_bwd_kernel<GtF32><<<gb, 256, 0, st>>>(img, b, W, H, maps, lambda, 0, grad, &sums[1]);
    }
}

// Sum of squared differences (for PSNR, metrics.cpp:91-101), FP64 per block.
template <typename Gt>
__global__ void __launch_bounds__(256) sqdiff_kernel(const float* __restrict__ a, const Gt b, int64_t n,
                                                     double* __restrict__ sum) {
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double d = (double)a[i] - (double)b[i];
        acc += d * d;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        atomicAdd(sum, t);
    }
}

// metrics of img against gt: sums[0] = SSIM sum over the valid positions and
// channels, sums[1] = sum of squared differences
void launch_metrics(cudaStream_t st, const float* img, const void* gt, bool gt_u8, int W, int H, float* maps,
                    double* sums) {
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    dim3 g((vw + 31) / 32, (vh + 31) / 32, 3);
    const int64_t n = (int64_t)W * H * 3;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 1184);
    if (gt_u8) {
        const GtU8 b{static_cast<const uint8_t*>(gt)};
        if (vw > 0 && vh > 0) ssim_fwd_kernel<GtU8><<<g, 256, 0, st>>>(img, b, W, H, maps, &sums[0]);
        sqdiff_kernel<GtU8><<<blocks, 256, 0, st>>>(img, b, n, &sums[1]);
    } else {
        const GtF32 b{static_cast<const float*>(gt)};
        if (vw > 0 && vh > 0) ssim_fwd_kernel<GtF32><<<g, 256, 0, st>>>(img, b, W, H, maps, &sums[0]);
        sqdiff_kernel<GtF32><<<blocks, 256, 0, st>>>(img, b, n, &sums[1]);
    }
}

}  // namespace hgs
