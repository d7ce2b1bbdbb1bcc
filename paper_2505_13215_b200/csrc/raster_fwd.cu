// raster_fwd.cu -- K2 (sorted-splat gather + tile-key duplication), tile
// ranges, K4 (tile rasterizer forward) and the FP64 fix-up pass.
//
// Reference: raster.cpp:167-235 (rasterize), 123-148 (composite_pixel),
// backward.cpp:142-175 (the taped forward, which must match bitwise).
#include "raster_common.cuh"

namespace hgs {

// After the depth sort: gather the exact record into depth order, derive the
// FP32 fast view (Cholesky of the scaled conic + certified error bound), and
// emit the tile count of each sorted splat.
__global__ void __launch_bounds__(256) gather_sorted_kernel(const uint32_t* __restrict__ sorted_gid, int V,
                                                            const SplatRec* __restrict__ rec,
                                                            const uint32_t* __restrict__ ntiles,
                                                            SplatRec* __restrict__ rec_sorted,
                                                            SplatFast* __restrict__ fast_sorted,
                                                            uint32_t* __restrict__ ntiles_sorted) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    const uint32_t gid = sorted_gid[j];
    const SplatRec e = rec[gid];
    rec_sorted[j] = e;
    ntiles_sorted[j] = ntiles[gid];
    SplatFast f;
    f.sx_hi = __double2float_rn(e.sx);
    f.sx_lo = __double2float_rn(e.sx - (double)f.sx_hi);
    f.sy_hi = __double2float_rn(e.sy);
    f.sy_lo = __double2float_rn(e.sy - (double)f.sy_hi);
    // x = power*log2e = d^T (0.5*log2e*Csym) d = |L d|^2, L upper triangular
    const double s = 0.5 * kLog2eD;
    const double a00 = s * e.c00, a01 = s * 0.5 * (e.c01 + e.c10), a11 = s * e.c11;
    bool fp64 = false;
    double l00 = 0.0, l01 = 0.0, l11 = 0.0;
    if (a00 > 0.0) {
        l00 = sqrt(a00);
        l01 = a01 / l00;
        const double rem = a11 - l01 * l01;
        if (rem > 0.0) l11 = sqrt(rem);
        else fp64 = true;
    } else {
        fp64 = true;
    }
    const double r = fp64 ? 1e30 : fabs(l01) / l11;
    if (r > 4.0) fp64 = true;
    f.l00 = (float)l00;
    f.l01 = (float)l01;
    f.l11 = (float)l11;
    f.alpha_f = e.alpha_f;
    f.r = e.r;
    f.g = e.g;
    f.b = e.b;
    // FP32 path: |x_f - x| <= u*X*(17 + 16r) over the relevant region x <= 8,
    // u = 2^-24 (two extra roundings for the double-float mean); relative
    // alpha error = ln2*|dx| + 2^-22 (ex2.approx) + 2 roundings.
    f.eps = fp64 ? 1.0e-6f : (float)(8.0e-6 * (1.0 + r) + 4.0e-7);
    f.x0 = e.x0;
    f.x1 = e.x1;
    f.y0 = e.y0;
    f.y1 = e.y1;
    f.fp64 = fp64 ? 1u : 0u;
    f.pad_ = 0u;
    fast_sorted[j] = f;
}

// Duplicate each sorted splat into every tile its box overlaps
// (raster.cpp:182-201); key = tile id, value = sorted splat index.
__global__ void __launch_bounds__(256) duplicate_kernel(const SplatFast* __restrict__ fast, int V,
                                                        const uint32_t* __restrict__ offsets, int tiles_x,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= V) return;
    const SplatFast f = fast[j];
    uint32_t o = offsets[j];
    const int tx0 = f.x0 / kTile, tx1 = f.x1 / kTile, ty0 = f.y0 / kTile, ty1 = f.y1 / kTile;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            keys[o] = (uint32_t)(ty * tiles_x + tx);
            vals[o] = (uint32_t)j;
            ++o;
        }
}

// Per-tile [start, end) into the tile-sorted instance list (raster.cpp:205-212).
__global__ void __launch_bounds__(256) tile_ranges_kernel(const uint32_t* __restrict__ keys, int n,
                                                          uint2* __restrict__ ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

constexpr int kBatch = 256;

// K4: one CTA per 16x16 tile, one thread per pixel, front-to-back alpha
// blending over the tile's depth-ordered list staged through shared memory in
// batches of 256 splats; CTA-wide early exit once every pixel saturated.
//
// Outputs per pixel: rgb (HWC float), last[pix] = one past the instance index
// of the last contributor (bit 31 = pixel handed to the FP64 fix-up), and the
// optional count / transmittance maps.
__global__ void __launch_bounds__(256) raster_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val, const SplatFast* __restrict__ fast,
    const SplatRec* __restrict__ exact, int W, int H, int tiles_x, float bg_r, float bg_g, float bg_b,
    float* __restrict__ out_rgb, uint32_t* __restrict__ out_last, float* __restrict__ out_tfinal,
    float* __restrict__ out_trans, uint32_t* __restrict__ out_count, uint32_t* __restrict__ fix_list,
    uint32_t* __restrict__ fix_count) {
    __shared__ SplatFast s_fast[kBatch];
    __shared__ uint32_t s_j[kBatch];
    const int tile = blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    const int px = tx * kTile + (threadIdx.x & 15);
    const int py = ty * kTile + (threadIdx.x >> 4);
    const bool inside = px < W && py < H;
    const uint2 rg = ranges[tile];
    const float pxc = (float)px + 0.5f, pyc = (float)py + 0.5f;
    const double pcx = (double)px + 0.5, pcy = (double)py + 0.5;

    float T = 1.0f, cr = 0.0f, cg = 0.0f, cb = 0.0f;
    float err = 0.0f;  // certified relative error bound of T
    uint32_t last = rg.x, count = 0;
    bool done = !inside, flagged = false;

    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t idx = base + threadIdx.x;
        if (idx < rg.y) {
            const uint32_t j = inst_val[idx];
            s_fast[threadIdx.x] = fast[j];
            s_j[threadIdx.x] = j;
        }
        __syncthreads();
        const int nb = min((uint32_t)kBatch, rg.y - base);
        for (int k = 0; k < nb && !done; ++k) {
            const SplatFast& f = s_fast[k];
            if (px < f.x0 || px > f.x1 || py < f.y0 || py > f.y1) continue;
            ++count;
            const float x = pair_x(f, exact[s_j[k]], pxc, pyc, pcx, pcy);
            float g;
            const float a = pair_alpha(f, exact[s_j[k]], x, pcx, pcy, g);
            if (a < 0.0f) continue;
            const float w = a * T;
            cr = fmaf(f.r, w, cr);
            cg = fmaf(f.g, w, cg);
            cb = fmaf(f.b, w, cb);
            const float om = 1.0f - a;
            err += __fdividef(a * f.eps, om) + 2.5e-7f;
            T *= om;
            last = base + k + 1;
            if (T < 1.0e-4f * (1.0f + 2.0f * err)) {
                // inside the error band of the oracle's T < 1e-4 decision?
                if (T > 1.0e-4f * (1.0f - 2.0f * err)) flagged = true;
                done = true;
            }
        }
    }
    if (!inside) return;
    const int pix = py * W + px;
    out_rgb[pix * 3 + 0] = fmaf(T, bg_r, cr);
    out_rgb[pix * 3 + 1] = fmaf(T, bg_g, cg);
    out_rgb[pix * 3 + 2] = fmaf(T, bg_b, cb);
    out_last[pix] = last | (flagged ? 0x80000000u : 0u);
    out_tfinal[pix] = T;
    if (out_trans) out_trans[pix] = T;
    if (out_count) out_count[pix] = count;
    if (flagged) fix_list[atomicAdd(fix_count, 1u)] = (uint32_t)pix;
}

// Exact FP64 recomposite of flagged pixels (raster.cpp:123-148 verbatim),
// one thread per pixel, grid-stride over the device-side count.
__global__ void __launch_bounds__(128) raster_fixup_kernel(
    const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ fix_count, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r,
    double bg_g, double bg_b, float* __restrict__ out_rgb, uint32_t* __restrict__ out_last,
    float* __restrict__ out_tfinal, float* __restrict__ out_trans, uint32_t* __restrict__ out_count) {
    const uint32_t n = *fix_count;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int pix = (int)fix_list[q];
        const int px = pix % W, py = pix / W;
        const int tile = (py / kTile) * tiles_x + px / kTile;
        const uint2 rg = ranges[tile];
        const double pcx = px + 0.5, pcy = py + 0.5;
        double T = 1.0, ar = 0.0, ag = 0.0, ab = 0.0;
        uint32_t count = 0, last = rg.x;
        for (uint32_t i = rg.x; i < rg.y; ++i) {
            const SplatRec& e = exact[inst_val[i]];
            if (px < e.x0 || px > e.x1 || py < e.y0 || py > e.y1) continue;
            ++count;
            const double a = __dmul_rn(e.alpha, exp(-exact_power(e, pcx, pcy)));
            if (a < kAlphaCutoff) continue;
            const double w = __dmul_rn(a, T);
            ar = __dadd_rn(ar, __dmul_rn((double)e.r, w));
            ag = __dadd_rn(ag, __dmul_rn((double)e.g, w));
            ab = __dadd_rn(ab, __dmul_rn((double)e.b, w));
            T = __dmul_rn(T, __dsub_rn(1.0, a));
            last = i + 1;
            if (T < kTransFloor) break;
        }
        out_rgb[pix * 3 + 0] = (float)__dadd_rn(ar, __dmul_rn(T, bg_r));
        out_rgb[pix * 3 + 1] = (float)__dadd_rn(ag, __dmul_rn(T, bg_g));
        out_rgb[pix * 3 + 2] = (float)__dadd_rn(ab, __dmul_rn(T, bg_b));
        out_last[pix] = last | 0x80000000u;
        out_tfinal[pix] = (float)T;
        if (out_trans) out_trans[pix] = (float)T;
        if (out_count) out_count[pix] = count;
    }
}

}  // namespace hgs
