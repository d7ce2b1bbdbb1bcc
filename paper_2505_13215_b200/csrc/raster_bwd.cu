// raster_bwd.cu -- K6: tile rasterizer backward (backward.cpp:178-222).
//
// One CTA per tile, one thread per pixel, re-evaluating every pair with the
// same arithmetic as K4 (so every contribute/skip decision is reproduced).
// Like the reference it walks each pixel's list BACK TO FRONT from the
// forward's recorded last contributor, accumulating the suffix colour
// S_i = sum_{j>i} c_j a_j T_j + T_final*bg by addition (accurate for deep,
// nearly occluded splats, unlike C_out - prefix) and recovering
// T_i = T_{i+1} / (1 - a_i) from the stored final transmittance.
//
// Per splat and warp the 9 accumulators are reduced with a transposing
// butterfly (14 shuffles instead of 45), summed across warps with shared
// atomics, and flushed once per tile batch with vector red.global.add.
// Pixels the forward handed to the FP64 fix-up are back-propagated by
// raster_bwd_exact_kernel (one warp per pixel, FP64).
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
    __shared__ SplatBatch<kBatchB> sb;
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
    // accumulates c_j a_j T_j from the back; T_i = T_{i+1} / (1 - a_i).
    float Sr = T * bg_r, Sg = T * bg_g, Sb = T * bg_b;
    const int nbatch = (int)((end - rg.x + kBatchB - 1) / kBatchB);
    for (int bi = nbatch - 1; bi >= 0; --bi) {
        const uint32_t base = rg.x + (uint32_t)bi * kBatchB;
        const int nb = (int)min((uint32_t)kBatchB, end - base);
        if ((int)threadIdx.x < nb) {
            const uint32_t j = inst_val[base + threadIdx.x];
            sb.load(threadIdx.x, fast, j);
            const SplatRec& e = exact[j];
            s_conic[threadIdx.x] = make_float4((float)e.c00, (float)e.c01, (float)e.c10, (float)e.c11);
        }
#pragma unroll
        for (int q = 0; q < kAccStride - 3; ++q) s_acc[threadIdx.x][q] = 0.f;
        __syncthreads();
        for (int k = nb - 1; k >= 0; --k) {
            float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            float v8 = 0.f;
            bool contrib = false;
            const int4 hdr = sb.hdr[k];
            if (base + k < last && in_box(hdr.x, hdr.y, px, py)) {
                float x, dx, dy;
                if (hdr.z) {
                    x = exact_x(exact + sb.j[k], pcx, pcy);
                    const float2 d = exact_delta(exact + sb.j[k], pcx, pcy);
                    dx = d.x;
                    dy = d.y;
                } else {
                    x = fast_x(sb.mean[k], sb.chol[k], pxc, pyc, dx, dy);
                }
                const float4 L = sb.chol[k];
                float g;
                const float a = pair_alpha(L.w, __int_as_float(hdr.w), x, exact + sb.j[k], pcx, pcy, g);
                if (a >= 0.0f) {
                    contrib = true;
                    const float4 col = sb.col[k];
                    const float inv = __frcp_rn(1.0f - a);
                    const float Ti = T * inv;  // transmittance before this splat
                    const float w = a * Ti;
                    // d_a = g_pix . (rgb * T_i - S / (1 - a))
                    const float d_a = gr * fmaf(col.x, Ti, -Sr * inv) + gg * fmaf(col.y, Ti, -Sg * inv) +
                                      gb * fmaf(col.z, Ti, -Sb * inv);
                    Sr = fmaf(col.x, w, Sr);
                    Sg = fmaf(col.y, w, Sg);
                    Sb = fmaf(col.z, w, Sb);
                    T = Ti;
                    v[0] = w * gr;
                    v[1] = w * gg;
                    v[2] = w * gb;
                    v[3] = g * d_a;
                    const float gdg = g * (L.w * d_a);  // g * d_g, d_g = alpha * d_a
                    const float4 c = s_conic[k];
                    v[4] = gdg * fmaf(c.x, dx, c.y * dy);
                    v[5] = gdg * fmaf(c.z, dx, c.w * dy);
                    const float hc = -0.5f * gdg;
                    v[6] = hc * dx * dx;
                    v[7] = hc * dx * dy;
                    v8 = hc * dy * dy;
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
                float* dst = accum + (size_t)sb.j[threadIdx.x] * kAccStride;
                red_add_v4(dst, a[0], a[1], a[2], a[3]);
                red_add_v4(dst + 4, a[4], a[5], a[6], a[7]);
                atomicAdd(dst + 8, a[8]);
            }
        }
        __syncthreads();
    }
}

// FP64 backward of the fix-up pixels (backward.cpp:182-221), one warp per
// pixel.  Pass 1 recomposites the pixel exactly like raster_fixup_kernel to
// get C_out; pass 2 walks the same list again: lanes evaluate 32 splats in
// parallel, the uniform sequential walk hands every contributing lane its
// T_i and inclusive prefix P_i, and the lanes then emit their gradient
// contributions with d_a = g.(c T_i - (C_out - P_i)/(1 - a)) (in FP64 the
// subtraction is exact enough) via global atomics.
__global__ void __launch_bounds__(128) raster_bwd_exact_kernel(
    const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ fix_count, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r,
    double bg_g, double bg_b, const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg,
    float* __restrict__ accum) {
    const uint32_t n = *fix_count;
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += warps) {
        const int pix = (int)fix_list[q];
        const double gp[3] = {dL_dimg[pix * 3], dL_dimg[pix * 3 + 1], dL_dimg[pix * 3 + 2]};
        if (gp[0] == 0.0 && gp[1] == 0.0 && gp[2] == 0.0) continue;
        const int px = pix % W, py = pix / W;
        const uint2 rg = ranges[(py / kTile) * tiles_x + px / kTile];
        const uint32_t last = last_arr[pix] & 0x7fffffffu;
        const double pcx = px + 0.5, pcy = py + 0.5;
        double Cout[3];
        for (int pass = 0; pass < 2; ++pass) {
            double T = 1.0, P[3] = {0.0, 0.0, 0.0};
            for (uint32_t base = rg.x; base < last; base += 32) {
                const uint32_t i = base + lane;
                double a = -1.0, g = 0.0;
                double rgb[3] = {0.0, 0.0, 0.0};
                const SplatRec* e = nullptr;
                if (i < last) {
                    e = &exact[inst_val[i]];
                    if (px >= e->x0 && px <= e->x1 && py >= e->y0 && py <= e->y1) {
                        g = exp(-exact_power(*e, pcx, pcy));
                        a = __dmul_rn(e->alpha, g);
                        rgb[0] = e->r;
                        rgb[1] = e->g;
                        rgb[2] = e->b;
                    }
                }
                const bool mine = a >= kAlphaCutoff;
                const unsigned cm = __ballot_sync(0xffffffffu, mine);
                double myT = 0.0, myP[3] = {0.0, 0.0, 0.0};
                for (int jj = 0; jj < 32; ++jj) {
                    if (!((cm >> jj) & 1u)) continue;
                    const double aj = __shfl_sync(0xffffffffu, a, jj);
                    const double w = aj * T;
                    for (int c = 0; c < 3; ++c) P[c] += __shfl_sync(0xffffffffu, rgb[c], jj) * w;
                    if (lane == jj) {
                        myT = T;
                        myP[0] = P[0];
                        myP[1] = P[1];
                        myP[2] = P[2];
                    }
                    T *= 1.0 - aj;
                }
                if (pass == 1 && mine) {
                    double d_a = 0.0;
                    for (int c = 0; c < 3; ++c) d_a += gp[c] * (rgb[c] * myT - (Cout[c] - myP[c]) / (1.0 - a));
                    float* dst = accum + (size_t)inst_val[i] * kAccStride;
                    const double w = a * myT;
                    for (int c = 0; c < 3; ++c) atomicAdd(dst + c, (float)(w * gp[c]));
                    atomicAdd(dst + 3, (float)(g * d_a));
                    const double d_g = e->alpha * d_a;
                    const double dx = pcx - e->sx, dy = pcy - e->sy;
                    const double q0 = e->c00 * dx + e->c01 * dy, q1 = e->c10 * dx + e->c11 * dy;
                    atomicAdd(dst + 4, (float)(g * d_g * q0));
                    atomicAdd(dst + 5, (float)(g * d_g * q1));
                    const double f = -0.5 * g * d_g;
                    atomicAdd(dst + 6, (float)(f * dx * dx));
                    atomicAdd(dst + 7, (float)(f * dx * dy));
                    atomicAdd(dst + 8, (float)(f * dy * dy));
                }
            }
            if (pass == 0) {
                Cout[0] = P[0] + T * bg_r;
                Cout[1] = P[1] + T * bg_g;
                Cout[2] = P[2] + T * bg_b;
            }
        }
    }
}

}  // namespace hgs
