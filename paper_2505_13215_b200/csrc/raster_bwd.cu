// raster_bwd.cu -- K6: tile rasterizer backward (backward.cpp:178-222).
//
// One CTA per tile, one thread per pixel, re-evaluating every pair with the
// same arithmetic as K4 (so every contribute/skip decision is reproduced; the
// walk is bounded by the forward's
// recorded last contributor).  Like the reference it walks each pixel's list
// BACK TO FRONT from the forward's last contributor, accumulating the suffix
// colour S_i = sum_{j>i} c_j a_j T_j + T_final*bg by addition (accurate for
// deep, nearly occluded splats, unlike C_out - prefix) and recovering
// T_i = T_{i+1} / (1 - a_i) from the stored final transmittance.
//
// Per splat and warp the 9 accumulators are reduced with a transposing
// butterfly (14 shuffles instead of 45), summed across warps with shared
// atomics, and flushed once per tile batch with vector red.global.add.
// Pixels the forward handed to the FP64 fix-up are back-propagated by
// raster_bwd_exact_kernel with the oracle's own reverse sweep.
#include "kernels.cuh"

namespace hgs {

namespace {

constexpr int kBatchB = 256;

// Transposing warp reduction of 8 values: afterwards lane L holds the warp
// total of value (L >> 2) (every lane of each group of four).
__device__ __forceinline__ float transpose_reduce8(float v[8]) {
    const int lane = threadIdx.x & 31;
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    float a4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = b4 ? v[k] : v[4 + k];
        const float keep = b4 ? v[4 + k] : v[k];
        a4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float a2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = b3 ? a4[k] : a4[2 + k];
        const float keep = b3 ? a4[2 + k] : a4[k];
        a2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float a1;
    {
        const float send = b2 ? a2[0] : a2[1];
        const float keep = b2 ? a2[1] : a2[0];
        a1 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
    a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
    return a1;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

}  // namespace

// accum layout: 12 floats per sorted splat (16-byte aligned for v4 reds):
//   [0..2] d_rgb, [3] d_alpha (w.r.t. the base alpha), [4..5] d_screen,
//   [6] d_conic00, [7] d_conic01 (= d_conic10), [8] d_conic11, [9..11] pad
constexpr int kAccStride = 12;

__global__ void __launch_bounds__(256) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val, const SplatFast* __restrict__ fast,
    const SplatRec* __restrict__ exact, int W, int H, int tiles_x, const float* __restrict__ tfinal,
    const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg, float bg_r, float bg_g, float bg_b,
    float* __restrict__ accum) {
    __shared__ SplatFast s_fast[kBatchB];
    __shared__ uint32_t s_j[kBatchB];
    __shared__ float4 s_conic[kBatchB];  // float conic (c00, c01, c10, c11)
    __shared__ float s_acc[kBatchB][kAccStride - 3];
    __shared__ uint32_t s_maxlast;
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const uint2 rg = ranges[tile];
    const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;
    const double pcx = (double)px + 0.5, pcy = (double)py + 0.5;

    uint32_t last = rg.x;
    float gr = 0.f, gg = 0.f, gb = 0.f, T = 1.f;
    if (inside) {
        const int pix = py * W + px;
        const uint32_t l = last_arr[pix];
        gr = dL_dimg[pix * 3 + 0];
        gg = dL_dimg[pix * 3 + 1];
        gb = dL_dimg[pix * 3 + 2];
        T = tfinal[pix];
        // flagged pixels go through the exact kernel; zero gradient = untouched (backward.cpp:188)
        if (!(l & 0x80000000u) && (gr != 0.f || gg != 0.f || gb != 0.f)) last = l;
    }
    if (threadIdx.x == 0) s_maxlast = rg.x;
    __syncthreads();
    if (last > rg.x) atomicMax(&s_maxlast, last);
    __syncthreads();
    const uint32_t end = s_maxlast;

    // Reverse sweep (backward.cpp:204-221): suffix S starts at T_final * bg and
    // accumulates c_j a_j T_j from the back, so it stays accurate relative to
    // its own (possibly tiny) magnitude; T_i = T_{i+1} / (1 - a_i).
    float Sr = T * bg_r, Sg = T * bg_g, Sb = T * bg_b;
    const int nbatch = (int)((end - rg.x + kBatchB - 1) / kBatchB);
    for (int bi = nbatch - 1; bi >= 0; --bi) {
        const uint32_t base = rg.x + (uint32_t)bi * kBatchB;
        const int nb = (int)min((uint32_t)kBatchB, end - base);
        if ((int)threadIdx.x < nb) {
            const uint32_t j = inst_val[base + threadIdx.x];
            s_fast[threadIdx.x] = fast[j];
            const SplatRec& e = exact[j];
            s_j[threadIdx.x] = j;
            s_conic[threadIdx.x] = make_float4((float)e.c00, (float)e.c01, (float)e.c10, (float)e.c11);
        }
#pragma unroll
        for (int q = 0; q < kAccStride - 3; ++q) s_acc[threadIdx.x][q] = 0.f;
        __syncthreads();
        for (int k = nb - 1; k >= 0; --k) {
            const uint32_t gidx = base + k;
            float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            float v8 = 0.f;
            bool contrib = false;
            if (gidx < last) {
                const SplatFast& f = s_fast[k];
                if (!(px < f.x0 || px > f.x1 || py < f.y0 || py > f.y1)) {
                    const float x = pair_x(f, exact[s_j[k]], pxc, pyc, pcx, pcy);
                    float g;
                    const float a = pair_alpha(f, exact[s_j[k]], x, pcx, pcy, g);
                    if (a >= 0.0f) {
                        contrib = true;
                        const float inv = __frcp_rn(1.0f - a);
                        const float Ti = T * inv;  // transmittance before this splat
                        const float w = a * Ti;
                        // d_a = g_pix . (rgb * T_i - S / (1 - a))
                        const float d_a = gr * fmaf(f.r, Ti, -Sr * inv) + gg * fmaf(f.g, Ti, -Sg * inv) +
                                          gb * fmaf(f.b, Ti, -Sb * inv);
                        Sr = fmaf(f.r, w, Sr);
                        Sg = fmaf(f.g, w, Sg);
                        Sb = fmaf(f.b, w, Sb);
                        T = Ti;
                        v[0] = w * gr;
                        v[1] = w * gg;
                        v[2] = w * gb;
                        v[3] = g * d_a;
                        const float d_g = f.alpha_f * d_a;
                        float dx, dy;
                        if (f.fp64) {
                            dx = (float)__dsub_rn(pcx, exact[s_j[k]].sx);
                            dy = (float)__dsub_rn(pcy, exact[s_j[k]].sy);
                        } else {
                            dx = __fsub_rn(__fsub_rn(pxc, f.sx_hi), f.sx_lo);
                            dy = __fsub_rn(__fsub_rn(pyc, f.sy_hi), f.sy_lo);
                        }
                        const float4 c = s_conic[k];
                        const float gdg = g * d_g;
                        v[4] = gdg * fmaf(c.x, dx, c.y * dy);
                        v[5] = gdg * fmaf(c.z, dx, c.w * dy);
                        const float hc = -0.5f * gdg;
                        v[6] = hc * dx * dx;
                        v[7] = hc * dx * dy;
                        v8 = hc * dy * dy;
                    }
                }
            }
            if (__any_sync(0xffffffffu, contrib)) {
                const float r8 = transpose_reduce8(v);
                const float r9 = warp_sum(v8);
                const int lane = threadIdx.x & 31;
                if ((lane & 3) == 0) atomicAdd(&s_acc[k][lane >> 2], r8);
                if (lane == 1) atomicAdd(&s_acc[k][8], r9);
            }
        }
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            const float* a = s_acc[threadIdx.x];
            bool nz = false;
#pragma unroll
            for (int q = 0; q < 9; ++q) nz |= a[q] != 0.f;
            if (nz) {
                float* dst = accum + (size_t)s_j[threadIdx.x] * kAccStride;
                red_add_v4(dst, a[0], a[1], a[2], a[3]);
                red_add_v4(dst + 4, a[4], a[5], a[6], a[7]);
                atomicAdd(dst + 8, a[8]);
            }
        }
        __syncthreads();
    }
}

// FP64 backward of the fix-up pixels: the oracle's per-pixel forward
// recompute and reverse suffix sweep (backward.cpp:182-221), scattered with
// atomics.  A handful of pixels per frame.
__global__ void __launch_bounds__(128) raster_bwd_exact_kernel(
    const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ fix_count, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r,
    double bg_g, double bg_b, const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg,
    float* __restrict__ accum) {
    const uint32_t n = *fix_count;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int pix = (int)fix_list[q];
        const double gp[3] = {dL_dimg[pix * 3], dL_dimg[pix * 3 + 1], dL_dimg[pix * 3 + 2]};
        if (gp[0] == 0.0 && gp[1] == 0.0 && gp[2] == 0.0) continue;
        const int px = pix % W, py = pix / W;
        const uint2 rg = ranges[(py / kTile) * tiles_x + px / kTile];
        const uint32_t last = last_arr[pix] & 0x7fffffffu;
        const double pcx = px + 0.5, pcy = py + 0.5;
        // forward recompute: final transmittance over the contributor list
        double T = 1.0;
        for (uint32_t i = rg.x; i < last; ++i) {
            const SplatRec& e = exact[inst_val[i]];
            if (px < e.x0 || px > e.x1 || py < e.y0 || py > e.y1) continue;
            const double a = __dmul_rn(e.alpha, exp(-exact_power(e, pcx, pcy)));
            if (a < kAlphaCutoff) continue;
            T = __dmul_rn(T, __dsub_rn(1.0, a));
        }
        // reverse sweep; T_i recovered by walking forward again per step is
        // O(n^2) -- instead store nothing and re-derive T_i = prod_{j<i}(1-a_j)
        // with a second forward pass that keeps a running suffix via the
        // identity S_i = C_out - P_i evaluated in double.
        double Cout[3];
        {
            double P[3] = {0, 0, 0}, Ti = 1.0;
            for (uint32_t i = rg.x; i < last; ++i) {
                const SplatRec& e = exact[inst_val[i]];
                if (px < e.x0 || px > e.x1 || py < e.y0 || py > e.y1) continue;
                const double a = __dmul_rn(e.alpha, exp(-exact_power(e, pcx, pcy)));
                if (a < kAlphaCutoff) continue;
                const double w = a * Ti;
                P[0] += (double)e.r * w;
                P[1] += (double)e.g * w;
                P[2] += (double)e.b * w;
                Ti *= 1.0 - a;
            }
            Cout[0] = P[0] + T * bg_r;
            Cout[1] = P[1] + T * bg_g;
            Cout[2] = P[2] + T * bg_b;
        }
        double P[3] = {0, 0, 0}, Ti = 1.0;
        for (uint32_t i = rg.x; i < last; ++i) {
            const uint32_t j = inst_val[i];
            const SplatRec& e = exact[j];
            if (px < e.x0 || px > e.x1 || py < e.y0 || py > e.y1) continue;
            const double pw = exact_power(e, pcx, pcy);
            const double g = exp(-pw);
            const double a = __dmul_rn(e.alpha, g);
            if (a < kAlphaCutoff) continue;
            const double rgb[3] = {e.r, e.g, e.b};
            const double w = a * Ti;
            for (int c = 0; c < 3; ++c) P[c] += rgb[c] * w;
            double d_a = 0.0;
            for (int c = 0; c < 3; ++c) d_a += gp[c] * (rgb[c] * Ti - (Cout[c] - P[c]) / (1.0 - a));
            float* dst = accum + (size_t)j * kAccStride;
            for (int c = 0; c < 3; ++c) atomicAdd(dst + c, (float)(w * gp[c]));
            atomicAdd(dst + 3, (float)(g * d_a));
            const double d_g = e.alpha * d_a;
            const double dx = pcx - e.sx, dy = pcy - e.sy;
            const double q0 = e.c00 * dx + e.c01 * dy, q1 = e.c10 * dx + e.c11 * dy;
            atomicAdd(dst + 4, (float)(g * d_g * q0));
            atomicAdd(dst + 5, (float)(g * d_g * q1));
            const double f = -0.5 * g * d_g;
            atomicAdd(dst + 6, (float)(f * dx * dx));
            atomicAdd(dst + 7, (float)(f * dx * dy));
            atomicAdd(dst + 8, (float)(f * dy * dy));
            Ti *= 1.0 - a;
        }
    }
}

}  // namespace hgs
