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
#include "kernels.cuh"

namespace hgs {

namespace {

constexpr int kWin = 11, kHalf = 5;
constexpr int kTX = 32, kTY = 16;  // outputs per CTA
constexpr int kSX = kTX + 2 * kHalf, kSY = kTY + 2 * kHalf;

__constant__ float c_win[kWin];

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

// grid: (ceil(vw/32), ceil(vh/16), 3 channels); block 256.
// a, b: HWC float images.  Writes maps (3 x planes of vw*vh per channel) and
// the per-block SSIM sums.
__global__ void __launch_bounds__(256) ssim_fwd_kernel(const float* __restrict__ a, const float* __restrict__ b, int W,
                                                       int H, float* __restrict__ maps, double* __restrict__ ssim_sum) {
    __shared__ float sa[kSY][kSX], sb[kSY][kSX];
    __shared__ float h[5][kSY][kTX];
    __shared__ float red[8];
    const int c = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
    for (int e = threadIdx.x; e < kSX * kSY; e += blockDim.x) {
        const int lx = e % kSX, ly = e / kSX;
        const int x = ox + lx, y = oy + ly;
        float va = 0.f, vb = 0.f;
        if (x < W && y < H) {
            va = a[((size_t)y * W + x) * 3 + c];
            vb = b[((size_t)y * W + x) * 3 + c];
        }
        sa[ly][lx] = va;
        sb[ly][lx] = vb;
    }
    __syncthreads();
    // horizontal pass: for each of the kSY rows and kTX output columns
    for (int e = threadIdx.x; e < kSY * kTX; e += blockDim.x) {
        const int lx = e % kTX, ly = e / kTX;
        float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
#pragma unroll
        for (int j = 0; j < kWin; ++j) {
            const float w = c_win[j];
            const float va = sa[ly][lx + j], vb = sb[ly][lx + j];
            m0 = fmaf(w, va, m0);
            m1 = fmaf(w, vb, m1);
            m2 = fmaf(w * va, va, m2);
            m3 = fmaf(w * vb, vb, m3);
            m4 = fmaf(w * va, vb, m4);
        }
        h[0][ly][lx] = m0;
        h[1][ly][lx] = m1;
        h[2][ly][lx] = m2;
        h[3][ly][lx] = m3;
        h[4][ly][lx] = m4;
    }
    __syncthreads();
    float local = 0.f;
    for (int e = threadIdx.x; e < kTX * kTY; e += blockDim.x) {
        const int lx = e % kTX, ly = e / kTX;
        const int vx = ox + lx, vy = oy + ly;
        if (vx >= vw || vy >= vh) continue;
        float mu_a = 0.f, mu_b = 0.f, aa = 0.f, bb = 0.f, ab = 0.f;
#pragma unroll
        for (int i = 0; i < kWin; ++i) {
            const float w = c_win[i];
            mu_a = fmaf(w, h[0][ly + i][lx], mu_a);
            mu_b = fmaf(w, h[1][ly + i][lx], mu_b);
            aa = fmaf(w, h[2][ly + i][lx], aa);
            bb = fmaf(w, h[3][ly + i][lx], bb);
            ab = fmaf(w, h[4][ly + i][lx], ab);
        }
        const float C1 = 1e-4f, C2 = 9e-4f;
        const float var_a = aa - mu_a * mu_a, var_b = bb - mu_b * mu_b, cov = ab - mu_a * mu_b;
        const float a1 = 2.f * mu_a * mu_b + C1, a2 = 2.f * cov + C2;
        const float b1 = mu_a * mu_a + mu_b * mu_b + C1, b2 = var_a + var_b + C2;
        const float denom = b1 * b2;
        const float s = a1 * a2 / denom;
        local += s;
        const float d_mu = (a2 / denom) * 2.f * mu_b - (s / b1) * 2.f * mu_a;
        const float d_var = -s / b2;
        const float d_cov = 2.f * a1 / denom;
        const size_t plane = (size_t)vw * vh;
        const size_t o = (size_t)c * 3 * plane + (size_t)vy * vw + vx;
        maps[o] = d_mu - 2.f * d_var * mu_a - d_cov * mu_b;
        maps[o + plane] = d_var;
        maps[o + 2 * plane] = d_cov;
    }
    const float tot = block_sum(local, red);
    if (threadIdx.x == 0) atomicAdd(ssim_sum, (double)tot);
}

// grid: (ceil(W/32), ceil(H/16), 3); dL/dimage = (1-l) sign(a-b)/n - l dSSIM/da.
__global__ void __launch_bounds__(256) ssim_bwd_kernel(const float* __restrict__ a, const float* __restrict__ b, int W,
                                                       int H, const float* __restrict__ maps, float lambda,
                                                       int with_ssim, float* __restrict__ grad,
                                                       double* __restrict__ l1_sum) {
    __shared__ float sm[3][kSY][kSX];
    __shared__ float h[3][kSY][kTX];
    __shared__ float red[8];
    const int c = blockIdx.z;
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const int ox = blockIdx.x * kTX, oy = blockIdx.y * kTY;
    const size_t plane = with_ssim ? (size_t)vw * vh : 0;
    if (with_ssim) {
        // maps at valid positions (x - 10 .. x) contribute to pixel x
        for (int e = threadIdx.x; e < kSX * kSY; e += blockDim.x) {
            const int lx = e % kSX, ly = e / kSX;
            const int vx = ox + lx - 2 * kHalf, vy = oy + ly - 2 * kHalf;
            float m0 = 0.f, m1 = 0.f, m2 = 0.f;
            if (vx >= 0 && vy >= 0 && vx < vw && vy < vh) {
                const size_t o = (size_t)c * 3 * plane + (size_t)vy * vw + vx;
                m0 = maps[o];
                m1 = maps[o + plane];
                m2 = maps[o + 2 * plane];
            }
            sm[0][ly][lx] = m0;
            sm[1][ly][lx] = m1;
            sm[2][ly][lx] = m2;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < kSY * kTX; e += blockDim.x) {
            const int lx = e % kTX, ly = e / kTX;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
            for (int j = 0; j < kWin; ++j) {
                // pixel x gets window weight w[x - vx] from the map at vx
                const float w = c_win[kWin - 1 - j];
                s0 = fmaf(w, sm[0][ly][lx + j], s0);
                s1 = fmaf(w, sm[1][ly][lx + j], s1);
                s2 = fmaf(w, sm[2][ly][lx + j], s2);
            }
            h[0][ly][lx] = s0;
            h[1][ly][lx] = s1;
            h[2][ly][lx] = s2;
        }
        __syncthreads();
    }
    const float inv_n = 1.0f / (float)((size_t)W * H * 3);
    const float inv_nv = with_ssim ? 1.0f / (float)((size_t)vw * vh * 3) : 0.f;
    float local = 0.f;
    for (int e = threadIdx.x; e < kTX * kTY; e += blockDim.x) {
        const int lx = e % kTX, ly = e / kTX;
        const int x = ox + lx, y = oy + ly;
        if (x >= W || y >= H) continue;
        const size_t p = ((size_t)y * W + x) * 3 + c;
        const float va = a[p], vb = b[p];
        const float d = va - vb;
        local += fabsf(d);
        float gsum = (1.0f - lambda) * ((d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) * inv_n);
        if (with_ssim) {
            float g0 = 0.f, g1 = 0.f, g2 = 0.f;
#pragma unroll
            for (int i = 0; i < kWin; ++i) {
                const float w = c_win[kWin - 1 - i];
                g0 = fmaf(w, h[0][ly + i][lx], g0);
                g1 = fmaf(w, h[1][ly + i][lx], g1);
                g2 = fmaf(w, h[2][ly + i][lx], g2);
            }
            const float dssim = (g0 + 2.f * va * g1 + vb * g2) * inv_nv;
            gsum -= lambda * dssim;
        }
        grad[p] = gsum;
    }
    const float tot = block_sum(local, red);
    if (threadIdx.x == 0) atomicAdd(l1_sum, (double)tot);
}

}  // namespace hgs
