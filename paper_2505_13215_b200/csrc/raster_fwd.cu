// raster_fwd.cu -- K2 (sorted-splat gather + tile-key duplication), tile
// culling and ranges, K4 (tile rasterizer forward) and the FP64 fix-up pass.
//
// Reference: raster.cpp:167-235 (rasterize), 123-148 (composite_pixel),
// backward.cpp:142-175 (the taped forward, which must match bitwise).
#include "kernels.cuh"

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
    // culling threshold on the power: alpha * exp(-p) >= 1/255  <=>  p <= ln(255 alpha)
    f.pcut = (float)(log(e.alpha * 255.0) + 1e-5);
    // FP32 path: |x_f - x| <= u*X*(17 + 16r) over the relevant region x <= 8,
    // u = 2^-24 (two extra roundings for the double-float mean); relative
    // alpha error = ln2*|dx| + 2^-22 (ex2.approx) + 2 roundings.
    f.eps = fp64 ? 1.0e-6f : (float)(8.0e-6 * (1.0 + r) + 4.0e-7);
    f.xr = (int32_t)e.x0 | ((int32_t)(e.x1 - e.x0) << 16);
    f.yr = (int32_t)e.y0 | ((int32_t)(e.y1 - e.y0) << 16);
    f.fp64 = fp64 ? 1u : 0u;
    fast_sorted[j] = f;
}

// Can splat e reach alpha >= 1/255 at any pixel centre of [xa,xb]x[ya,yb]?
// Minimum of the (convex) power over the rectangle: 0 if the mean is inside,
// else on one of the four edges at the clamped 1D minimiser, compared with
// pcut = ln(alpha * 255) + 1e-5 (a 1e-5 margin on the power, i.e. ~1e-5
// relative on alpha).  A pair skipped here is one the reference skips too
// (raster.cpp:139-140), so the output is unchanged.
__device__ inline bool tile_may_contribute(const SplatRec& e, double pcut, int xa, int xb, int ya, int yb) {
    const double lx = xa + 0.5 - e.sx, hx = xb + 0.5 - e.sx, ly = ya + 0.5 - e.sy, hy = yb + 0.5 - e.sy;
    if (lx <= 0.0 && 0.0 <= hx && ly <= 0.0 && 0.0 <= hy) return true;
    const double a = e.c00, b = 0.5 * (e.c01 + e.c10), c = e.c11;
    auto q = [&](double dx, double dy) { return 0.5 * (a * dx * dx + 2.0 * b * dx * dy + c * dy * dy); };
    double pmin = INFINITY;
    const double xs[2] = {lx, hx}, ys[2] = {ly, hy};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const double dy = fmin(fmax(-b * xs[k] / c, ly), hy);
        pmin = fmin(pmin, q(xs[k], dy));
        const double dx = fmin(fmax(-b * ys[k] / a, lx), hx);
        pmin = fmin(pmin, q(dx, ys[k]));
    }
    return pmin <= pcut;
}

// Duplicate each sorted splat into every tile its box overlaps
// (raster.cpp:182-201), one thread per INSTANCE (binary search of the splat
// in the exclusive tile-count scan) so splats covering hundreds of tiles do
// not serialise; key = tile id, value = sorted splat index with bit 31 set
// when the splat cannot reach the alpha cutoff anywhere in that tile.
__global__ void __launch_bounds__(256) duplicate_kernel(const SplatFast* __restrict__ fast,
                                                        const SplatRec* __restrict__ exact, int V,
                                                        const uint32_t* __restrict__ offsets, int tiles_x, int cull,
                                                        uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                        int I) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= I) return;
    int lo = 0, hi = V - 1;  // last j with offsets[j] <= i
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&offsets[mid]) <= (uint32_t)i) lo = mid;
        else hi = mid - 1;
    }
    const int j = lo;
    const int32_t xr = __ldg(&fast[j].xr), yr = __ldg(&fast[j].yr);
    const int x0 = box_x0(xr), x1 = x0 + box_w(xr), y0 = box_x0(yr), y1 = y0 + box_w(yr);
    const int tx0 = x0 / kTile, tx1 = x1 / kTile, ty0 = y0 / kTile;
    const int local = i - (int)__ldg(&offsets[j]);
    const int w = tx1 - tx0 + 1;
    const int ty = ty0 + local / w, tx = tx0 + local % w;
    uint32_t v = (uint32_t)j;
    if (cull && !(tx0 == tx1 && ty0 == y1 / kTile)) {
        const double pcut = (double)__ldg(&fast[j].pcut);
        if (!tile_may_contribute(exact[j], pcut, max(x0, tx * kTile), min(x1, tx * kTile + kTile - 1),
                                 max(y0, ty * kTile), min(y1, ty * kTile + kTile - 1)))
            v |= 0x80000000u;
    }
    keys[i] = (uint32_t)(ty * tiles_x + tx);
    vals[i] = v;
}

__global__ void __launch_bounds__(256) keep_flag_kernel(const uint32_t* __restrict__ vals, int n,
                                                        uint32_t* __restrict__ flag) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (vals[i] >> 31) ? 0u : 1u;
}

// Stable compaction of the tile-sorted instances that can contribute.
__global__ void __launch_bounds__(256) compact_instances_kernel(const uint32_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ vals, int n,
                                                                const uint32_t* __restrict__ pos,
                                                                uint32_t* __restrict__ keys_out,
                                                                uint32_t* __restrict__ vals_out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t v = vals[i];
    if (v >> 31) return;
    const uint32_t p = pos[i];
    keys_out[p] = keys[i];
    vals_out[p] = v;
}

// Per-tile [start, end) into a tile-sorted instance list (raster.cpp:205-212).
__global__ void __launch_bounds__(256) tile_ranges_kernel(const uint32_t* __restrict__ keys, int n,
                                                          uint2* __restrict__ ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

__global__ void __launch_bounds__(256) tile_ranges_dev_kernel(const uint32_t* __restrict__ keys,
                                                              const uint32_t* __restrict__ n_dev,
                                                              uint2* __restrict__ ranges) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = (int)*n_dev;
    if (i >= n) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

constexpr int kBatch = 256;

// K4: one CTA per 16x16 tile, one thread per pixel, front-to-back alpha
// blending over the tile's depth-ordered list staged through shared memory
// (SoA, LDS.128 broadcasts) in batches of 256 splats; CTA-wide early exit once
// every pixel saturated.
//
// Outputs per pixel: rgb (HWC float), last[pix] = one past the instance index
// of the last contributor (bit 31 = pixel handed to the FP64 fix-up), the
// final transmittance (read by the backward) and the optional count /
// transmittance maps.
__global__ void __launch_bounds__(256) raster_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val, const SplatFast* __restrict__ fast,
    const SplatRec* __restrict__ exact, int W, int H, int tiles_x, float bg_r, float bg_g, float bg_b,
    float* __restrict__ out_rgb, uint32_t* __restrict__ out_last, float* __restrict__ out_tfinal,
    float* __restrict__ out_trans, uint32_t* __restrict__ out_count, uint32_t* __restrict__ fix_list,
    uint32_t* __restrict__ fix_count) {
    __shared__ SplatBatch<kBatch> sb;
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
        if (idx < rg.y) sb.load(threadIdx.x, fast, inst_val[idx]);
        __syncthreads();
        const int nb = min((uint32_t)kBatch, rg.y - base);
        for (int k = 0; k < nb && !done; ++k) {
            const int4 hdr = sb.hdr[k];
            if (!in_box(hdr.x, hdr.y, px, py)) continue;
            ++count;
            float x, dx, dy;
            if (hdr.z) x = exact_x(exact + sb.j[k], pcx, pcy);
            else x = fast_x(sb.mean[k], sb.chol[k], pxc, pyc, dx, dy);
            const float4 L = sb.chol[k];
            const float eps = __int_as_float(hdr.w);
            float g;
            const float a = pair_alpha(L.w, eps, x, exact + sb.j[k], pcx, pcy, g);
            if (a < 0.0f) continue;
            const float4 c = sb.col[k];
            const float w = a * T;
            cr = fmaf(c.x, w, cr);
            cg = fmaf(c.y, w, cg);
            cb = fmaf(c.z, w, cb);
            const float om = 1.0f - a;
            err += __fdividef(a * eps, om) + 2.5e-7f;
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

// Exact FP64 recomposite of the flagged pixels (raster.cpp:123-148), one warp
// per pixel: the 32 lanes evaluate 32 consecutive splats' box test and FP64
// alpha in parallel, then every lane walks them in order (uniform loop) to
// apply the oracle's sequential transmittance update and break.
__global__ void __launch_bounds__(128) raster_fixup_kernel(
    const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ fix_count, const uint2* __restrict__ ranges,
    const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r,
    double bg_g, double bg_b, float* __restrict__ out_rgb, uint32_t* __restrict__ out_last,
    float* __restrict__ out_tfinal, float* __restrict__ out_trans, uint32_t* __restrict__ out_count) {
    const uint32_t n = *fix_count;
    const int lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < n; q += warps) {
        const int pix = (int)fix_list[q];
        const int px = pix % W, py = pix / W;
        const uint2 rg = ranges[(py / kTile) * tiles_x + px / kTile];
        const double pcx = px + 0.5, pcy = py + 0.5;
        double T = 1.0, ar = 0.0, ag = 0.0, ab = 0.0;
        uint32_t count = 0, last = rg.x;
        bool done = false;
        for (uint32_t base = rg.x; base < rg.y && !done; base += 32) {
            const uint32_t i = base + lane;
            bool inb = false;
            double a = -1.0, r = 0.0, g = 0.0, b = 0.0;
            if (i < rg.y) {
                const SplatRec& e = exact[inst_val[i]];
                inb = px >= e.x0 && px <= e.x1 && py >= e.y0 && py <= e.y1;
                if (inb) {
                    a = exact_alpha(e, pcx, pcy);
                    r = e.r;
                    g = e.g;
                    b = e.b;
                }
            }
            const unsigned inmask = __ballot_sync(0xffffffffu, inb);
            const int cnt = (int)min(32u, rg.y - base);
            for (int jj = 0; jj < cnt; ++jj) {
                if (!((inmask >> jj) & 1u)) continue;
                ++count;
                const double aj = __shfl_sync(0xffffffffu, a, jj);
                if (aj < kAlphaCutoff) continue;
                const double rj = __shfl_sync(0xffffffffu, r, jj), gj = __shfl_sync(0xffffffffu, g, jj),
                             bj = __shfl_sync(0xffffffffu, b, jj);
                const double w = __dmul_rn(aj, T);
                ar = __dadd_rn(ar, __dmul_rn(rj, w));
                ag = __dadd_rn(ag, __dmul_rn(gj, w));
                ab = __dadd_rn(ab, __dmul_rn(bj, w));
                T = __dmul_rn(T, __dsub_rn(1.0, aj));
                last = base + jj + 1;
                if (T < kTransFloor) {
                    done = true;
                    break;
                }
            }
        }
        if (lane == 0) {
            out_rgb[pix * 3 + 0] = (float)__dadd_rn(ar, __dmul_rn(T, bg_r));
            out_rgb[pix * 3 + 1] = (float)__dadd_rn(ag, __dmul_rn(T, bg_g));
            out_rgb[pix * 3 + 2] = (float)__dadd_rn(ab, __dmul_rn(T, bg_b));
            out_last[pix] = last | 0x80000000u;
            out_tfinal[pix] = (float)T;
            if (out_trans) out_trans[pix] = (float)T;
            if (out_count) out_count[pix] = count;
        }
    }
}

}  // namespace hgs
