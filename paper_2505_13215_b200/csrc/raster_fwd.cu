// raster_fwd.cu -- K2 (sorted-splat gather + tile-key duplication), tile
// culling and ranges, K4 (tile rasterizer forward) and the FP64 fix-up pass.
//
// Reference: raster.cpp:167-235 (rasterize), 123-148 (composite_pixel),
// backward.cpp:142-175 (the taped forward, which must match bitwise).
#include <cstddef>

#include "kernels.cuh"

namespace hgs {

// Diagnostics only (HGS_DEBUG_EXACT, read at context creation; 0 in every
// measured or tested configuration): bit 0 -- every splat takes the FP64
// exponent path; bit 1 -- every pixel goes through the FP64 fix-up (forward)
// and exact backward.
__device__ int g_debug_exact = 0;
__device__ float g_debug_terr = INFINITY;  // HGS_DEBUG_TERR: flag pixels whose T error bound exceeds it

void set_debug_exact(int v) { cudaMemcpyToSymbol(g_debug_exact, &v, sizeof(int)); }
void set_debug_terr(float v) { cudaMemcpyToSymbol(g_debug_terr, &v, sizeof(float)); }

// After the depth sort: gather the exact record into depth order, derive the
// FP32 fast view (Cholesky of the scaled conic + certified error bound), and
// emit the tile count of each sorted splat.
__device__ inline void band_terms(CullRec& e);  // (below, with the band test)

__global__ void __launch_bounds__(256) gather_sorted_kernel(const uint32_t* __restrict__ sorted_gid,
                                                            const uint32_t* __restrict__ V_dev,
                                                            const SplatRec* __restrict__ rec,
                                                            const uint32_t* __restrict__ ntiles,
                                                            SplatRec* __restrict__ rec_sorted,
                                                            SplatFast* __restrict__ fast_sorted,
                                                            uint32_t* __restrict__ ntiles_sorted,
                                                            uint32_t* __restrict__ sorted_of_gid,
                                                            CullRec* __restrict__ cull_rec) {
    pdl_wait();  // launched with launch_pdl
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (int)*V_dev) return;
    const uint32_t gid = sorted_gid[j];
    if (sorted_of_gid) sorted_of_gid[gid] = (uint32_t)j;  // (null: no backward of this render)
    const SplatRec e = rec[gid];
    if (rec_sorted) rec_sorted[j] = e;  // (null: sweep frame without a tape; K4 reads rec via the depth order)
    // tile culling (FP32, conservative): threshold on the power, alpha * exp(-p)
    // >= 1/255 <=> p <= ln(255 alpha) (+1e-5 margin, see tile_may_contribute)
    {
        CullRec cr;
        cr.sx_hi = __double2float_rn(e.sx);
        cr.sx_lo = __double2float_rn(e.sx - (double)cr.sx_hi);
        cr.sy_hi = __double2float_rn(e.sy);
        cr.sy_lo = __double2float_rn(e.sy - (double)cr.sy_hi);
        cr.a = (float)e.c00;
        cr.b = (float)(0.5 * (e.c01 + e.c10));
        cr.c = (float)e.c11;
        cr.pcut = (float)(log(e.alpha * 255.0) + 1e-5);
        band_terms(cr);
        cull_rec[j] = cr;
    }
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
    if (r > 16.0) fp64 = true;  // FP32 stays certified (e1 grows with r); measured best at 16
    if (g_debug_exact & 1) fp64 = true;
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
    // The error of x grows with x itself: |x_f - x| <= u*x*(17 + 16r), i.e. a
    // relative alpha error <= e1*x + e0 with e1 = ln2*u*(17 + 16r) <=
    // 1e-6*(1 + r) and e0 = 4e-7 (FP64 path: x only rounded, e1 = 1e-7).
    // The cutoff guard band uses the bound at x <= 8; the transmittance
    // error (K4) uses the per-pair bound, tight for the opaque core.
    const double e1 = fp64 ? 1.0e-7 : 1.0e-6 * (1.0 + r);
    const double eps = 8.0 * e1 + 4.0e-7;
    cutoff_thresholds((double)e.alpha_f, eps, f.x_skip, f.x_keep);
    f.eps = fp64 ? -(float)e1 : (float)e1;  // sign bit selects the FP64 exponent path
    f.xr = (int32_t)e.x0 | ((int32_t)(e.x1 - e.x0) << 16);
    f.yr = (int32_t)e.y0 | ((int32_t)(e.y1 - e.y0) << 16);
    fast_sorted[j] = f;
}

// Can splat e reach alpha >= 1/255 at any pixel centre of [xa,xb]x[ya,yb]?
// Minimum of the (convex) power over the rectangle: 0 if the mean is inside,
// else on one of the four edges at the clamped 1D minimiser, compared with
// pcut = ln(alpha * 255) + 1e-5.  Evaluated in FP32 and CONSERVATIVE: the
// rectangle is declared unreachable only when the FP32 minimum exceeds pcut
// by more than its error bound (1e-5 of the summed magnitudes S of the
// quadratic's terms, >> the ~10 ulp actual error, plus 1e-5 absolute), so a
// pair skipped here is one the reference skips too (raster.cpp:139-140) and
// the output is unchanged; doubtful rectangles are simply kept.
__device__ inline bool tile_may_contribute(const CullRec& e, int xa, int xb, int ya, int yb) {
    const float lx = fast_dx((float)xa + 0.5f, e.sx_hi, e.sx_lo), hx = fast_dx((float)xb + 0.5f, e.sx_hi, e.sx_lo);
    const float ly = fast_dx((float)ya + 0.5f, e.sy_hi, e.sy_lo), hy = fast_dx((float)yb + 0.5f, e.sy_hi, e.sy_lo);
    if (lx <= 0.0f && 0.0f <= hx && ly <= 0.0f && 0.0f <= hy) return true;
    const float a = e.a, b = e.b, c = e.c;
    if (!(a > 0.0f && c > 0.0f)) return true;  // not positive definite in FP32: keep
    const float ia = __fdividef(1.0f, a), ic = __fdividef(1.0f, c);  // minimiser only: approximate is fine
    float pmin = INFINITY, smag = 0.0f;
    auto eval = [&](float dx, float dy) {
        const float bxy = b * dx * dy;
        const float q = 0.5f * fmaf(a * dx, dx, fmaf(c * dy, dy, 2.0f * bxy));
        if (q < pmin) {
            pmin = q;
            smag = 0.5f * fmaf(a * dx, dx, fmaf(c * dy, dy, 2.0f * fabsf(bxy)));
        }
    };
    const float xs[2] = {lx, hx}, ys[2] = {ly, hy};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        eval(xs[k], fminf(fmaxf(-b * xs[k] * ic, ly), hy));
        eval(fminf(fmaxf(-b * ys[k] * ia, lx), hx), ys[k]);
    }
    return pmin <= e.pcut + 1e-5f * (1.0f + smag);
}

// The same question for the four 8x8 quadrants of a tile at once, through
// the ellipse E = {power <= pcut} itself: for each quadrant row (band of
// pixel-centre offsets dy in [y1, y2]) the x-range of E over the band is
// [XL, XR] -- the ellipse's own x-extreme +-X_ext when the extreme point's
// dy lies in the band, else the boundary at the nearer band edge (the
// right boundary is concave, the left convex, in dy) -- and a quadrant is
// reachable iff its x-range overlaps [XL, XR].  Same answer as
// tile_may_contribute (min of a convex function over a rectangle <= pcut
// <=> the rectangle meets E), a fraction of its arithmetic.  FP32 with
// margins covering its rounding: pcut + 1e-5 (1 + 2|pcut|); X_ext / Y_ext and
// the band clip widened by 1e-3 relative + 1e-3 px; XR / XL widened by
// 2e-3 (X_ext + |b| max|dy| / a) + 1e-3 px (the sqrt of a cancelling
// difference loses at most sqrt(8u) of the half-width).  Only for conics
// with det >= 1e-3 a c (well conditioned); otherwise (and for
// non-positive-definite or empty cases) returns false = "use the exact
// per-quadrant test".
// The splat's tile-independent terms of the band test (once per splat, in
// gather_sorted); X_ext < 0 marks conics the test does not apply to
// (non-positive-definite, ill-conditioned det < 1e-3 a c, empty E).
__device__ inline void band_terms(CullRec& e) {
    const float a = e.a, b = e.b, c = e.c;
    e.X_ext = -1.0f;
    if (!(a > 0.0f && c > 0.0f)) return;
    const float det = fmaf(a, c, -b * b);
    if (!(det >= 1e-3f * a * c)) return;
    const float P2 = 2.0f * (e.pcut + 1e-5f * (1.0f + 2.0f * fabsf(e.pcut)));
    if (!(P2 > 0.0f)) return;
    const float X_ext = sqrtf(P2 * c / det), Y_ext = sqrtf(P2 * a / det);
    e.X_ext = X_ext;
    e.Yc = Y_ext * 1.001f + 1e-3f;  // band clip (wider: conservative)
    e.dyr = -b * X_ext / c;         // dy of the rightmost point of E (leftmost: -dyr)
    e.inv_a = 1.0f / a;
    e.aP2 = a * P2;
    e.det = det;
    e.tol = 1e-3f * Y_ext + 1e-3f;
    e.mB = 2e-3f * fabsf(b) * e.inv_a;
}

__device__ inline bool quadrant_mask_bands(const CullRec& e, int x0, int x1, int y0, int y1, int tx, int ty,
                                           uint32_t& mask) {
    const float X_ext = e.X_ext;
    if (!(X_ext >= 0.0f)) return false;
    const float b = e.b, Yc = e.Yc, dyr = e.dyr, inv_a = e.inv_a, aP2 = e.aP2, det = e.det, tol = e.tol;
    mask = 0u;
#pragma unroll
    for (int qy = 0; qy < 2; ++qy) {
        const int ya = max(y0, ty * kTile + qy * 8), yb = min(y1, ty * kTile + qy * 8 + 7);
        if (ya > yb) continue;
        const float y1f = fast_dx((float)ya + 0.5f, e.sy_hi, e.sy_lo), y2f = fast_dx((float)yb + 0.5f, e.sy_hi, e.sy_lo);
        const float lo = fmaxf(y1f, -Yc), hi = fminf(y2f, Yc);
        if (lo > hi) continue;  // the band misses E
        float XR, XL;
        if (dyr >= lo - tol && dyr <= hi + tol) {
            XR = X_ext;
        } else {
            const float d = fminf(fmaxf(dyr, lo), hi);
            XR = (-b * d + sqrtf(fmaxf(0.0f, fmaf(-det * d, d, aP2)))) * inv_a;
        }
        if (-dyr >= lo - tol && -dyr <= hi + tol) {
            XL = -X_ext;
        } else {
            const float d = fminf(fmaxf(-dyr, lo), hi);
            XL = (-b * d - sqrtf(fmaxf(0.0f, fmaf(-det * d, d, aP2)))) * inv_a;
        }
        const float m = fmaf(e.mB, fmaxf(fabsf(lo), fabsf(hi)), 2e-3f * X_ext) + 1e-3f;
        XR += m;
        XL -= m;
#pragma unroll
        for (int qx = 0; qx < 2; ++qx) {
            const int xa = max(x0, tx * kTile + qx * 8), xb = min(x1, tx * kTile + qx * 8 + 7);
            if (xa > xb) continue;
            const float lx = fast_dx((float)xa + 0.5f, e.sx_hi, e.sx_lo), hx = fast_dx((float)xb + 0.5f, e.sx_hi, e.sx_lo);
            if (hx >= XL && lx <= XR) mask |= 1u << (qy * 2 + qx);
        }
    }
    return true;
}

// Duplicate each sorted splat into every tile its box overlaps
// (raster.cpp:182-201), one thread per INSTANCE so splats covering hundreds of
// tiles do not serialise.  A CTA covers kDupPerCta consecutive instances: two
// global binary searches bound its splat range [j_lo, j_hi] (at most
// kDupPerCta splats, every visible splat owns >= 1 instance), whose offsets
// are staged in shared memory for the per-instance searches.
// key = tile id, value = sorted splat index | 4-bit quadrant mask << 28.
constexpr int kDupThreads = 256, kDupPerCta = kDupPerCtaHost;

__device__ __forceinline__ int last_le(const uint32_t* __restrict__ off, int lo, int hi, uint32_t i) {
    while (lo < hi) {  // last j in [lo, hi] with off[j] <= i (off[lo] <= i)
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// cta_first[b] = the sorted splat owning instance b * kDupPerCta (each CTA
// boundary lies in exactly one splat's [offset, offset + ntiles) range).
// V_dev (optional): the visible count on the device (capacity-mode renders
// launch for N); nblocks bounds the writes (cta_first has nblocks + 1 entries:
// the CTAs of the capacity and the first splat past it).
__global__ void __launch_bounds__(256) dup_bounds_kernel(const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ ntiles_sorted, int V,
                                                         uint32_t* __restrict__ cta_first, const uint32_t* V_dev,
                                                         uint32_t nblocks, uint32_t* __restrict__ zero_words,
                                                         uint32_t n_zero) {
    pdl_wait();  // launched with launch_pdl
    // the look-back status words (+ tile counter) of duplicate_compact_kernel
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_zero; i += gridDim.x * blockDim.x)
        zero_words[i] = 0u;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= (V_dev ? (int)*V_dev : V)) return;
    const uint32_t o = offsets[j], n = ntiles_sorted[j];
    for (uint32_t b = (o + kDupPerCta - 1) / kDupPerCta; b * kDupPerCta < o + n && b <= nblocks; ++b)
        cta_first[b] = (uint32_t)j;
}

// One instance i of the CTA's range: tile key and value (sorted splat index |
// quadrant mask << 28).  s_off: the offsets of splats [j_lo, j_lo + cnt).
// instance i of the CTA's splat window; jl: the local index of its splat
// (the last staged offset <= i)
__device__ __forceinline__ void dup_instance_at(int i, int jl, const uint32_t* s_off, int cnt, int j_lo,
                                                const SplatFast* __restrict__ fast, int cull,
                                                const CullRec* __restrict__ cull_rec, int tiles_x, uint32_t& key,
                                                uint32_t& val) {
    HGS_DCHECK(jl >= 0 && jl < cnt);
    const int j = j_lo + jl;
    const int32_t xr = __ldg(&fast[j].xr), yr = __ldg(&fast[j].yr);
    const int x0 = box_x0(xr), x1 = x0 + box_w(xr), y0 = box_x0(yr), y1 = y0 + box_w(yr);
    const int tx0 = x0 / kTile, tx1 = x1 / kTile, ty0 = y0 / kTile;
    const int local = i - (int)s_off[jl];
    const int w = tx1 - tx0 + 1;
    const int ty = ty0 + local / w, tx = tx0 + local % w;
    // one bit per 8x8 quadrant of the tile (bit q = qy*2 + qx): can the splat
    // reach the cutoff at a pixel of quadrant q inside its box?  Each quadrant
    // is one warp of the rasterizers, so the test is warp-uniform there.
    uint32_t mask = 0xfu;
    if (cull) {
        const CullRec e = cull_rec[j];
        if (!quadrant_mask_bands(e, x0, x1, y0, y1, tx, ty, mask)) {
            mask = 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int qx0 = tx * kTile + (q & 1) * 8, qy0 = ty * kTile + (q >> 1) * 8;
                const int xa = max(x0, qx0), xb = min(x1, qx0 + 7), ya = max(y0, qy0), yb = min(y1, qy0 + 7);
                if (xa <= xb && ya <= yb && tile_may_contribute(e, xa, xb, ya, yb)) mask |= 1u << q;
            }
        }
    }
    key = (uint32_t)(ty * tiles_x + tx);
    val = (uint32_t)j | (mask << kInstMaskShift);
}

__device__ __forceinline__ void dup_instance(int i, const uint32_t* s_off, int cnt, int j_lo,
                                             const SplatFast* __restrict__ fast, int cull,
                                             const CullRec* __restrict__ cull_rec, int tiles_x, uint32_t& key,
                                             uint32_t& val) {
    dup_instance_at(i, last_le(s_off, 0, cnt - 1, (uint32_t)i), s_off, cnt, j_lo, fast, cull, cull_rec, tiles_x, key,
                    val);
}

__device__ __forceinline__ uint32_t dup_warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Duplication fused with the exact culling compaction: each CTA claims the
// next 1024-instance tile in order (atomic counter), evaluates its instances
// (4 consecutive per thread), block-scans the keep flags, obtains the number
// of kept instances before it by decoupled look-back over the earlier tiles,
// and writes only the kept (tile key, value) pairs -- in the reference's
// order, without materialising the full instance list.  status: one 64-bit
// (flag << 32 | count) word per tile, zeroed before the launch.
// (8 CTAs/SM, 32 registers: latency-bound on the per-instance loads and the
// look-back; full occupancy beats the spills -- -2% at c2 and c5 vs 48 registers)
__global__ void __launch_bounds__(kDupThreads, 8) duplicate_compact_kernel(
    const SplatFast* __restrict__ fast, int V, const uint32_t* __restrict__ offsets, int tiles_x,
    const CullRec* __restrict__ cull_rec, const uint32_t* __restrict__ cta_first, int I,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint32_t* __restrict__ kept_total,
    unsigned long long* status, uint32_t* __restrict__ counter, const uint32_t* V_dev, const uint32_t* I_dev,
    uint32_t* flags) {
    pdl_wait();  // launched with launch_pdl
    __shared__ uint32_t s_off[kDupPerCta + 1];
    __shared__ uint32_t s_tile, s_excl, s_wt[kDupThreads / 32];
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    // capacity mode (I_dev set): I is the launch capacity, the true count is on
    // the device; beyond the capacity the render is flagged (and redone by the host)
    if (V_dev) V = (int)*V_dev;
    int I_all = I;  // every instance (capacity mode: may exceed the launch capacity I)
    if (I_dev) {
        I_all = (int)*I_dev;
        if (I_all > I) {
            if (s_tile == 0 && threadIdx.x == 0) atomicOr(flags, FLAG_CAPACITY);
        } else {
            I = I_all;
        }
    }
    const int tile = (int)s_tile;
    const int i0 = tile * kDupPerCta;
    if (i0 >= I) return;  // CTAs of the capacity beyond the instances (nothing looks back at them)
    const int i_end = min(i0 + kDupPerCta, I);
    const int j_lo = (int)cta_first[tile];
    // the CTA's NOMINAL end decides whether cta_first[tile + 1] exists: in an
    // overflowing capacity-mode frame (I < I_all) i_end is clipped to the
    // capacity, but dup_bounds_kernel wrote only the boundaries below I_all
    const int j_hi = (tile + 1) * kDupPerCta < I_all ? (int)cta_first[tile + 1] : V - 1;
    const int cnt = min(j_hi - j_lo + 1, kDupPerCta + 1);  // a CTA spans at most kDupPerCta + 1 splats
    HGS_DCHECK(j_lo >= 0 && cnt >= 1 && j_lo + cnt <= V && (unsigned long long)V <= g_chk.splats);
    for (int k = threadIdx.x; k < cnt; k += kDupThreads) s_off[k] = __ldg(&offsets[j_lo + k]);
    __syncthreads();
    constexpr int kPer = kDupPerCta / kDupThreads;  // 4 consecutive instances per thread
    uint32_t key[kPer], val[kPer];
    uint32_t nk = 0;
    // one search for the thread's first instance, then forward steps (its
    // 4 consecutive instances span few splats)
    int jl = last_le(s_off, 0, cnt - 1, (uint32_t)min(i0 + (int)threadIdx.x * kPer, i_end - 1));
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const int i = i0 + threadIdx.x * kPer + k;
        key[k] = 0u;
        val[k] = 0u;
        if (i < i_end) {
            while (jl + 1 < cnt && s_off[jl + 1] <= (uint32_t)i) ++jl;
            dup_instance_at(i, jl, s_off, cnt, j_lo, fast, 1, cull_rec, tiles_x, key[k], val[k]);
        }
        nk += (val[k] >> kInstMaskShift) ? 1u : 0u;
    }
    // block exclusive scan of the kept counts
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t incl = dup_warp_incl_scan(nk);
    if (lane == 31) s_wt[warp] = incl;
    __syncthreads();
    uint32_t wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kDupThreads / 32; ++w) {
        const uint32_t x = s_wt[w];
        wbase += w < warp ? x : 0u;
        tot += x;
    }
    const uint32_t ex = wbase + incl - nk;
    if (threadIdx.x < 32) {
        // warp 0: publish the aggregate, look back 32 predecessors at a time.
        // Memory model: each status word carries its own payload (flag << 32 |
        // count) in one aligned 64-bit relaxed gpu-scope access -- single-copy
        // atomic, so a reader sees either 0 or a complete (flag, count); no
        // other data is published through it, so no acquire / release pairing
        // is needed.  Progress: tiles are claimed in launch order by the
        // atomic counter, so every predecessor is resident or finished.
        unsigned long long* st = status;
        uint32_t excl = 0;
        if (tile > 0) {
            if (lane == 0) st_relaxed_u64(st + tile, (1ull << 32) | tot);
            int hi = tile - 1;
            while (true) {
                const int p = hi - lane;
                unsigned long long w = p >= 0 ? ld_relaxed_u64(st + p) : (2ull << 32);
                uint32_t flag = (uint32_t)(w >> 32);
                while (__any_sync(0xffffffffu, flag == 0u)) {
                    if (flag == 0u) {
                        w = ld_relaxed_u64(st + p);
                        flag = (uint32_t)(w >> 32);
                    }
                }
                const unsigned pm = __ballot_sync(0xffffffffu, flag == 2u);
                const int stop = pm ? __ffs(pm) - 1 : 32;
                uint32_t v = (lane <= stop && p >= 0) ? (uint32_t)w : 0u;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (pm) break;
                hi -= 32;
            }
        }
        if (lane == 0) {
            st_relaxed_u64(st + tile, (2ull << 32) | (excl + tot));
            s_excl = excl;
            if (i_end >= I) *kept_total = excl + tot;
        }
    }
    __syncthreads();
    uint32_t pos = s_excl + ex;
#pragma unroll
    for (int k = 0; k < kPer; ++k)
        if (val[k] >> kInstMaskShift) {
            HGS_DCHECK(pos < (uint32_t)I && (unsigned long long)I <= g_chk.inst);
            keys_out[pos] = key[k];
            vals_out[pos] = val[k];
            ++pos;
        }
}

__global__ void __launch_bounds__(kDupThreads) duplicate_kernel(const SplatFast* __restrict__ fast,
                                                                const SplatRec* __restrict__ exact, int V,
                                                                const uint32_t* __restrict__ offsets, int tiles_x,
                                                                int cull, const CullRec* __restrict__ cull_rec,
                                                                uint32_t* __restrict__ keys,
                                                                uint32_t* __restrict__ vals,
                                                                uint32_t* __restrict__ keep,
                                                                const uint32_t* __restrict__ cta_first, int I) {
    __shared__ uint32_t s_off[kDupPerCta + 1];
    const int i0 = blockIdx.x * kDupPerCta;
    const int i_last = min(i0 + kDupPerCta, I) - 1;
    // splats [j_lo, j_hi] cover this CTA's instances (j_hi may own none of them)
    const int j_lo = (int)cta_first[blockIdx.x];
    const int j_hi = blockIdx.x + 1 < gridDim.x ? (int)cta_first[blockIdx.x + 1] : V - 1;
    const int cnt = j_hi - j_lo + 1;
    for (int k = threadIdx.x; k < cnt; k += kDupThreads) s_off[k] = __ldg(&offsets[j_lo + k]);
    __syncthreads();
    for (int i = i0 + threadIdx.x; i <= i_last; i += kDupThreads) {
        uint32_t key, val;
        dup_instance(i, s_off, cnt, j_lo, fast, cull, cull_rec, tiles_x, key, val);
        keys[i] = key;
        vals[i] = val;
        if (keep) keep[i] = (val >> kInstMaskShift) ? 1u : 0u;
    }
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
    if (!(v >> kInstMaskShift)) return;
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
    pdl_wait();  // launched with launch_pdl
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = (int)*n_dev;
    if (i >= n) return;
    const uint32_t t = keys[i];
    if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

// The rasterizers' launch order: tiles by descending instance count
// (counting sort on len / 8, capped; order within a bucket arbitrary), so the
// longest tiles start in the first wave and the last wave holds short ones
// (the tail of a K4 / K6 launch was ~5% of its duration).  One CTA.
// K6 uses the same order (ordering it by its own walk lengths, written by K4,
// measured 2% slower: the extra launch and a worse proxy).
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges, int n_tiles,
                                                          uint32_t* __restrict__ order) {
    pdl_wait();  // launched with launch_pdl
    __shared__ uint32_t hist[256];
    const int tid = threadIdx.x;
    if (tid < 256) hist[tid] = 0u;
    __syncthreads();
    auto bucket = [&](int t) {
        const uint2 r = ranges[t];
        return 255u - min((r.y - r.x) >> 3, 255u);  // heaviest first
    };
    for (int t = tid; t < n_tiles; t += blockDim.x) atomicAdd(&hist[bucket(t)], 1u);
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 256 buckets, 8 per lane
        uint32_t v[8], run = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            v[q] = hist[tid * 8 + q];
            run += v[q];
        }
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (tid >= o) incl += u;
        }
        uint32_t ex = incl - run;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            hist[tid * 8 + q] = ex;
            ex += v[q];
        }
    }
    __syncthreads();
    for (int t = tid; t < n_tiles; t += blockDim.x) order[atomicAdd(&hist[bucket(t)], 1u)] = (uint32_t)t;
}

constexpr int kBatch = 256;
constexpr int kThreads = 128;  // 16x16 tile, two pixels (rows y and y+8) per thread

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Exact FP64 recomposite of one flagged pixel (raster.cpp:123-148) by one
// warp over 32-splat chunks (exact_chunk: lane-parallel FP64 alphas, the
// transmittance chain in list order, colours summed lane-parallel in FP64).
// q: the pixel's fix-list slot (its FP64 colour goes to out_cout[q] for
// raster_bwd_exact_kernel).  Out of line: K4 calls it after its main loop.
static __device__ __noinline__ void fixup_pixel(uint32_t q, int pix, uint2 rg, const uint32_t* __restrict__ inst_val,
                                               const SplatRec* __restrict__ exact, const uint32_t* __restrict__ remap,
                                               int W, double bg_r, double bg_g,
                                               double bg_b, float* __restrict__ out_rgb, uint32_t* __restrict__ out_last,
                                               float* __restrict__ out_tfinal, float* __restrict__ out_trans,
                                               uint32_t* __restrict__ out_count, double* __restrict__ out_cout,
                                               double* s_om) {
    const int lane = threadIdx.x & 31;
    HGS_DCHECK(pix >= 0 && (unsigned long long)pix < g_chk.pixels);
    HGS_DCHECK(rg.x <= rg.y && rg.y <= g_chk.inst);
    const int px = pix % W, py = pix / W;
    const double pcx = px + 0.5, pcy = py + 0.5;
    double T = 1.0, ar = 0.0, ag = 0.0, ab = 0.0;
    uint32_t count = 0, last = rg.x;
    constexpr int S = kExactSub;
    for (uint32_t base = rg.x; base < rg.y; base += 32 * S) {
        ExactChunk<S> c;
        exact_chunk<S>(inst_val, exact, remap, base, rg.y, px, py, pcx, pcy, T, s_om, c);
        double wr = 0.0, wg = 0.0, wb = 0.0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            // in-box splats up to (and including) the terminating one
            const int tl = c.term - 32 * s;
            const uint32_t upto = (c.term < 0 || tl >= 31) ? 0xffffffffu : tl < 0 ? 0u : ((2u << tl) - 1u);
            count += __popc(c.inmask[s] & upto);
            if (c.contrib[s]) {
                const double w = __dmul_rn(c.a[s], c.Ti[s]);
                wr += c.e[s]->r * w;
                wg += c.e[s]->g * w;
                wb += c.e[s]->b * w;
            }
            const uint32_t cb = __ballot_sync(0xffffffffu, c.contrib[s]);
            if (cb) last = base + 32 * s + (31 - __clz(cb)) + 1;
        }
        ar += warp_sum_d(wr);
        ag += warp_sum_d(wg);
        ab += warp_sum_d(wb);
        if (c.term >= 0) break;
    }
    if (lane == 0) {
        const double cr = __dadd_rn(ar, __dmul_rn(T, bg_r)), cg = __dadd_rn(ag, __dmul_rn(T, bg_g)),
                     cb = __dadd_rn(ab, __dmul_rn(T, bg_b));
        out_rgb[pix * 3 + 0] = (float)cr;
        out_rgb[pix * 3 + 1] = (float)cg;
        out_rgb[pix * 3 + 2] = (float)cb;
        out_cout[3 * q + 0] = cr;
        out_cout[3 * q + 1] = cg;
        out_cout[3 * q + 2] = cb;
        out_last[pix] = last | 0x80000000u;
        out_tfinal[pix] = (float)T;
        if (out_trans) out_trans[pix] = (float)T;
        if (out_count) out_count[pix] = count;
    }
    __syncwarp();
}

// Per-pixel compositing state of K4.
struct PixFwd {
    float T, r, g, b, err;
    uint32_t last, count;
    bool done, flagged;
};

// The two pixels of a lane, packed (lo = row y, hi = row y + 4).  E is the
// certified ABSOLUTE error bound of T (|T_fp32 - T_oracle| <= E).  A pixel is
// finished exactly when T < 1e-4 + 2E (the certified band's upper edge): T
// and E change only on contributing pairs, so the test recomputed from the
// state equals the reference's break (raster.cpp:141-143); the pixel is
// flagged for the FP64 fix-up when its final T also lies above the band's
// lower edge 1e-4 - 2E.
struct PixFwd2 {
    f2 T, r, g, b, E;
    uint32_t last0, last1, count0, count1;
};

__device__ __forceinline__ f2 term_limit(const PixFwd2& s) { return f2_fma(f2_bc(2.0f), s.E, f2_bc(1.0e-4f)); }

// One pair of raster.cpp:132-143 for both pixels given their alphas (p0 / p1
// = the pixel's pair passes the 1/255 test; a no-op for that pixel
// otherwise).  Per pixel exactly the scalar sequence
//   w = a T; rgb += c w; T' = T (1 - a); E' = E (1 - a) + w eps + 2.5e-7 T'
// The error bound: with a_f = a (1 + d), |d| <= eps, and two roundings in
// fl(T fl(1 - a_f)),  T' - T'_oracle = (T - T_oracle)(1 - a) - T a d + 2u T',
// so E' above bounds it (2.5e-7 > 2u (1 + u) with u = 2^-24; the (1 - a_f)
// vs (1 - a) factor on E and E's own FP32 rounding are second order, inside
// that margin) -- the relative bound err of the earlier form times T, without
// its division by 1 - a.  A is exactly 0 for a pixel whose pair does not
// contribute (its exponent argument is replaced by 128: ex2.approx.ftz(-128)
// flushes to +0), so the updates are then exactly the identity (T * 1,
// E * 1 + 0 + 0, rgb + c * 0); only the rounding term needs the pass flag.
__device__ __forceinline__ void composite_pairs(PixFwd2& s, bool p0, bool p1, f2 A, f2 EPS, const float4 c,
                                                uint32_t idx) {
    const f2 AT = f2_mul(A, s.T);
    s.r = f2_fma(f2_bc(c.x), AT, s.r);
    s.g = f2_fma(f2_bc(c.y), AT, s.g);
    s.b = f2_fma(f2_bc(c.z), AT, s.b);
    const f2 OM = f2_sub(f2_bc(1.0f), A);
    const f2 TN = f2_mul(s.T, OM);
    const f2 U = f2_pk(p0 ? 2.5e-7f : 0.0f, p1 ? 2.5e-7f : 0.0f);
    s.E = f2_fma(s.E, OM, f2_fma(AT, EPS, f2_mul(TN, U)));
    s.T = TN;
    s.last0 = p0 ? idx + 1 : s.last0;
    s.last1 = p1 ? idx + 1 : s.last1;
}

__device__ __forceinline__ void write_pixel(const PixFwd& s, int pix, float bg_r, float bg_g, float bg_b,
                                            float* __restrict__ out_rgb, uint32_t* __restrict__ out_last,
                                            float* __restrict__ out_tfinal, float* __restrict__ out_trans,
                                            uint32_t* __restrict__ out_count, uint32_t* __restrict__ fix_list,
                                            uint32_t* __restrict__ fix_count, uint32_t* s_nfix, uint2* s_fix,
                                            uint32_t* __restrict__ fix_slot) {
    const bool flagged = s.flagged || (g_debug_exact & 2) || s.err > g_debug_terr * s.T;
    out_rgb[pix * 3 + 0] = fmaf(s.T, bg_r, s.r);
    out_rgb[pix * 3 + 1] = fmaf(s.T, bg_g, s.g);
    out_rgb[pix * 3 + 2] = fmaf(s.T, bg_b, s.b);
    out_last[pix] = s.last | (flagged ? 0x80000000u : 0u);
    out_tfinal[pix] = s.T;
    if (out_trans) out_trans[pix] = s.T;
    if (out_count) out_count[pix] = s.count;
    if (flagged) {  // the fix-list slot (the backward's exact pixels) and the CTA's own list
        const uint32_t q = atomicAdd(fix_count, 1u);
        fix_list[q] = (uint32_t)pix;
        fix_slot[pix] = q;  // K6 finds the pixel's FP64 colour through it
        s_fix[atomicAdd(s_nfix, 1u)] = make_uint2((uint32_t)pix, q);
    }
}

// K4: one CTA (128 threads) per 16x16 tile, two pixels per thread, front-to-
// back alpha blending over the tile's depth-ordered list staged through shared
// memory (SoA, LDS.128 broadcasts) in batches of 256 splats; CTA-wide early
// exit once every pixel saturated.  Each staged splat is read once for both
// pixels of a thread.
//
// Outputs per pixel: rgb (HWC float), last[pix] = one past the instance index
// of the last contributor (bit 31 = pixel handed to the FP64 fix-up), the
// final transmittance (read by the backward) and the optional count /
// transmittance maps.
template <bool kCount>  // kCount: per-pixel count of box-covered splats (count_map)
__global__ void __launch_bounds__(kThreads, 8) raster_fwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val, const SplatFast* __restrict__ fast,
    const SplatRec* __restrict__ exact, int W, int H, int tiles_x, float bg_r, float bg_g, float bg_b,
    float* __restrict__ out_rgb, uint32_t* __restrict__ out_last, float* __restrict__ out_tfinal,
    float* __restrict__ out_trans, uint32_t* __restrict__ out_count, uint32_t* __restrict__ fix_list,
    uint32_t* __restrict__ fix_count, const uint32_t* __restrict__ tile_order, double bg_rd, double bg_gd,
    double bg_bd, double* __restrict__ out_cout, uint32_t* __restrict__ fix_slot, const uint32_t* __restrict__ remap) {
    pdl_wait();  // launched with launch_pdl
    __shared__ SplatBatch<kBatch> sb;
    __shared__ uint32_t s_nfix;  // the CTA's pixels handed to the FP64 fix-up
    if (threadIdx.x == 0) s_nfix = 0u;
    __shared__ uint16_t s_list[kThreads / 32][kBatch];  // per-warp splat lists (build_warp_list)
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    // warp w owns the 8x8 quadrant (w & 1, w >> 1); a lane owns rows y, y+4
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py0 = ty * kTile + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
    const bool in0 = px < W && py0 < H, in1 = px < W && py1 < H;
    HGS_DCHECK((unsigned long long)tile < g_chk.tiles);
    const uint2 rg = ranges[tile];
    HGS_DCHECK(rg.x <= rg.y && rg.y <= g_chk.inst);
    const float pxc = (float)px + 0.5f, pyc0 = (float)py0 + 0.5f, pyc1 = (float)py1 + 0.5f;
    // FP64 pixel centres for the rare exact paths, rebuilt there (opaque: not
    // hoisted into 6 loop-carried registers of the 64)
    auto pcx = [&] { return (double)(int)opaque_u32((uint32_t)px) + 0.5; };
    auto pcy = [&](int py) { return (double)(int)opaque_u32((uint32_t)py) + 0.5; };

    // the box test's bits in a staged tile-relative mask (column bit | row bit):
    // a pixel is in the box iff both are set
    const int cshift = px - tx * kTile, rshift0 = 16 + py0 - ty * kTile;
    // per-thread loop constants in shared memory (read back with volatile
    // loads where needed): the box-test bits and the FP32 pixel-centre column
    __shared__ uint4 s_pix[kThreads];
    s_pix[threadIdx.x] = make_uint4((1u << cshift) | (1u << rshift0), (1u << cshift) | (1u << (rshift0 + 4)),
                                    __float_as_uint(pxc), 0u);
    const uint32_t a_pix = opaque_u32((uint32_t)__cvta_generic_to_shared(&s_pix[threadIdx.x]));
    PixFwd2 s;
    s.T = f2_bc(1.0f);
    s.r = s.g = s.b = s.E = f2_bc(0.0f);
    s.last0 = s.last1 = rg.x;
    s.count0 = s.count1 = 0u;
    const f2 PYC = f2_pk(pyc0, pyc1);
#ifdef HGS_CHECKED
    unsigned long long n_it = 0, n_box = 0, n_pass = 0, n_wit = 0;
#endif
    using SB = SplatBatch<kBatch>;
    const uint32_t sbase = opaque_u32((uint32_t)__cvta_generic_to_shared(&sb));
    const uint32_t a_bm = sbase + offsetof(SB, bm), a_hdr = sbase + offsetof(SB, hdr),
                   a_chol = sbase + offsetof(SB, chol), a_col = sbase + offsetof(SB, col),
                   a_mean = sbase + offsetof(SB, mean), a_j = sbase + offsetof(SB, j);

    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
        {
            const f2 LIM = term_limit(s);
            const bool act = (in0 && f2_lo(s.T) >= f2_lo(LIM)) || (in1 && f2_hi(s.T) >= f2_hi(LIM));
            if (__syncthreads_count(act) == 0) break;
        }
        for (int t = threadIdx.x; t < kBatch; t += kThreads) {
            const uint32_t idx = base + t;
            if (idx < rg.y) sb.load(t, fast, inst_val[idx], tx * kTile, ty * kTile);
        }
        __syncthreads();
        const int nb = min((uint32_t)kBatch, rg.y - base);
        // the splats whose quadrant-mask bit is set for this warp (exact: no
        // pixel of the quadrant reaches 1/255 otherwise)
        const int cnt = build_warp_list<kBatch>(sb.qm, sb.bm, nb, warp, s_list[warp]);
        const uint32_t a_list = opaque_u32((uint32_t)__cvta_generic_to_shared(&s_list[warp][0]));
#ifdef HGS_CHECKED
        n_wit += cnt;  // upper bound: the warp's list (lanes may finish earlier)
#endif
        // a lane leaves the walk once both its pixels finished (a per-lane exit:
        // warp-uniform votes here measured 3% slower)
        for (int q = 0; q < cnt; ++q) {
            const f2 LIM = term_limit(s);
            bool b0 = in0 && f2_lo(s.T) >= f2_lo(LIM), b1 = in1 && f2_hi(s.T) >= f2_hi(LIM);
            if (!(b0 || b1)) break;  // both pixels finished
#ifdef HGS_CHECKED
            if (b0 || b1) ++n_it;
#endif
            const uint32_t le = lds_u16(a_list + 2 * q);
            const uint32_t o16 = le & 0x0ff0u, o4 = o16 >> 2;
            const int k = (int)(o16 >> 4);
            const int4 hdr = lds_i4(a_hdr + o16);
            // box test: known true when the box covers the quadrant, else from
            // the staged tile-relative column/row masks
            if (!(le & 0x8000u)) {
                const uint32_t bm = lds_u32(a_bm + o4);
                const uint2 bx = ldsv_u2(a_pix);
                b0 = b0 && (bm & bx.x) == bx.x;
                b1 = b1 && (bm & bx.y) == bx.y;
                if (!(b0 || b1)) continue;
            }
            if (kCount) {
                s.count0 += b0;
                s.count1 += b1;
            }
#ifdef HGS_CHECKED
            n_box += (int)b0 + (int)b1;
#endif
            const float4 L = lds_f4(a_chol + o16), c = lds_f4(a_col + o16);
            // the exact record (rare paths only: loaded there)
            auto rec = [&] {
                const uint32_t j = lds_u32(a_j + o4);
                return exact + (remap ? __ldg(remap + j) : j);
            };
            const float eps_s = __int_as_float(hdr.w);
            // a pixel outside the box keeps x = 128: finite, so its EPS (and A * EPS
            // = 0 in composite_pairs) stays finite, and above every x_skip
            float x0 = 128.0f, x1 = 128.0f;
            if (eps_s < 0.0f) {  // FP64 exponent path (uniform per splat)
                if (b0) x0 = exact_x(rec(), pcx(), pcy(py0));
                if (b1) x1 = exact_x(rec(), pcx(), pcy(py1));
            } else {  // both pixels share the column: one dx, the rest packed (= fast_x per pixel)
                const float4 m = lds_f4(a_mean + o16);
                const float dx = __fsub_rn(__fsub_rn(ldsv_f(a_pix + 8), m.x), m.z);
                const f2 DY = f2_sub(f2_sub(PYC, f2_bc(m.y)), f2_bc(m.w));
                const f2 U1 = f2_fma(f2_bc(L.x), f2_bc(dx), f2_mul(f2_bc(L.y), DY));
                const f2 U2 = f2_mul(f2_bc(L.z), DY);
                const f2 X = f2_fma(U1, U1, f2_mul(U2, U2));
                x0 = f2_lo(X);
                x1 = f2_hi(X);
            }
            // the oracle's a >= 1/255 test (exact: FP64 inside the guard band)
            const float x_skip = __int_as_float(hdr.z), x_keep = c.w;
            bool p0 = b0 && x0 < x_skip, p1 = b1 && x1 < x_skip;
            const bool band0 = p0 && x0 >= x_keep, band1 = p1 && x1 >= x_keep;
            if (band0 || band1) {  // rare
                if (band0) p0 = exact_alpha_passes(rec(), pcx(), pcy(py0));
                if (band1) p1 = exact_alpha_passes(rec(), pcx(), pcy(py1));
            }
            if (!(p0 || p1)) continue;
#ifdef HGS_CHECKED
            n_pass += (int)p0 + (int)p1;
#endif
            const f2 X2 = f2_pk(x0, x1);
            const f2 A = f2_mul(f2_bc(L.w), f2_pk(fast_exp2_neg(p0 ? x0 : 128.0f), fast_exp2_neg(p1 ? x1 : 128.0f)));
            const f2 EPS = f2_fma(f2_bc(fabsf(eps_s)), X2, f2_bc(kAlphaErr0));
            composite_pairs(s, p0, p1, A, EPS, c, base + k);
        }
    }
#ifdef HGS_CHECKED
    HGS_COUNT_PAIRS(0, n_it);
    HGS_COUNT_PAIRS(1, n_box);
    HGS_COUNT_PAIRS(2, n_pass);
    if (lane == 0) HGS_COUNT_PAIRS(3, n_wit);
#endif
    // flagged: finished inside the certified error band of the T < 1e-4 decision
    const f2 LIM = term_limit(s), LOW = f2_fma(f2_bc(-2.0f), s.E, f2_bc(1.0e-4f));
    const bool flag0 = f2_lo(s.T) < f2_lo(LIM) && f2_lo(s.T) > f2_lo(LOW);
    const bool flag1 = f2_hi(s.T) < f2_hi(LIM) && f2_hi(s.T) > f2_hi(LOW);
    // after the walk the staged batch is dead: its memory holds the CTA's
    // fix-up list (hdr) and the fix-up walks' transmittance factors (mean)
    __syncthreads();
    uint2* s_fix = reinterpret_cast<uint2*>(&sb.hdr[0]);  // <= 256 entries (pixel, fix-list slot)
    if (in0) {
        const PixFwd s0{f2_lo(s.T), f2_lo(s.r), f2_lo(s.g), f2_lo(s.b), f2_lo(s.E), s.last0, s.count0, true,
                        flag0};
        write_pixel(s0, py0 * W + px, bg_r, bg_g, bg_b, out_rgb, out_last, out_tfinal, out_trans, out_count, fix_list,
                    fix_count, &s_nfix, s_fix, fix_slot);
    }
    if (in1) {
        const PixFwd s1{f2_hi(s.T), f2_hi(s.r), f2_hi(s.g), f2_hi(s.b), f2_hi(s.E), s.last1, s.count1, true,
                        flag1};
        write_pixel(s1, py1 * W + px, bg_r, bg_g, bg_b, out_rgb, out_last, out_tfinal, out_trans, out_count, fix_list,
                    fix_count, &s_nfix, s_fix, fix_slot);
    }
    // the FP64 fix-up of this tile's flagged pixels (~0.1% of the pixels), one
    // warp per pixel, inside the CTA: the walks overlap the other CTAs' work
    // instead of forming a serial tail kernel
    __syncthreads();
    const uint32_t nfix = s_nfix;
    double* s_om = reinterpret_cast<double*>(&sb.mean[0]) + warp * (32 * kExactSub);
    for (uint32_t k = warp; k < nfix; k += kThreads / 32) {
        const uint2 f = s_fix[k];
        fixup_pixel(f.y, (int)f.x, rg, inst_val, exact, remap, W, bg_rd, bg_gd, bg_bd, out_rgb, out_last, out_tfinal,
                    out_trans, out_count, out_cout, s_om);
    }
}

// Host launcher (keeps the template instantiations in this translation unit).
void launch_raster_fwd(bool count_map, int n_tiles, cudaStream_t st, const uint2* ranges, const uint32_t* inst_val,
                       const SplatFast* fast, const SplatRec* exact, int W, int H, int tiles_x, float bg_r, float bg_g,
                       float bg_b, float* out_rgb, uint32_t* out_last, float* out_tfinal, float* out_trans,
                       uint32_t* out_count, uint32_t* fix_list, uint32_t* fix_count, uint32_t* tile_order,
                       double bg_rd, double bg_gd, double bg_bd, double* out_cout, uint32_t* fix_slot,
                       const uint32_t* remap) {
    if (tile_order) {
        launch_pdl(tile_order_kernel, dim3(1), dim3(1024), 0, st, ranges, n_tiles, tile_order);
        count_launch();
    }
    const uint32_t* order = tile_order;
    if (count_map)
        launch_pdl(raster_fwd_kernel<true>, dim3(n_tiles), dim3(kThreads), 0, st, ranges, inst_val, fast, exact, W, H,
                   tiles_x, bg_r, bg_g, bg_b, out_rgb, out_last, out_tfinal, out_trans, out_count, fix_list,
                   fix_count, order, bg_rd, bg_gd, bg_bd, out_cout, fix_slot, remap);
    else
        launch_pdl(raster_fwd_kernel<false>, dim3(n_tiles), dim3(kThreads), 0, st, ranges, inst_val, fast, exact, W,
                   H, tiles_x, bg_r, bg_g, bg_b, out_rgb, out_last, out_tfinal, out_trans, out_count, fix_list,
                   fix_count, order, bg_rd, bg_gd, bg_bd, out_cout, fix_slot, remap);
}

// ---- density_map (raster.cpp:268-287)
__global__ void __launch_bounds__(256) density_diff_kernel(const uint32_t* __restrict__ ntiles,
                                                           const SplatRec* __restrict__ rec, int n, int W, int H,
                                                           int* __restrict__ diff) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || ntiles[i] == 0u) return;  // culled (not projected)
    const SplatRec& e = rec[i];
    const int x0 = e.x0, x1 = e.x1, y0 = e.y0, y1 = e.y1;
    atomicAdd(&diff[y0 * (W + 1) + x0], 1);
    atomicAdd(&diff[y0 * (W + 1) + x1 + 1], -1);
    atomicAdd(&diff[(y1 + 1) * (W + 1) + x0], -1);
    atomicAdd(&diff[(y1 + 1) * (W + 1) + x1 + 1], 1);
}

// inclusive prefix along each row (one warp per row)
__global__ void __launch_bounds__(256) density_rows_kernel(int* __restrict__ diff, int W, int H) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row > H) return;
    int* r = diff + (size_t)row * (W + 1);
    int carry = 0;
    for (int x0 = 0; x0 <= W; x0 += 32) {
        const int x = x0 + lane;
        int v = x <= W ? r[x] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (x <= W) r[x] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
}

// inclusive prefix down each column (one thread per column)
__global__ void __launch_bounds__(256) density_cols_kernel(const int* __restrict__ diff, int W, int H,
                                                           uint32_t* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= W) return;
    int acc = 0;
    for (int y = 0; y < H; ++y) {
        acc += diff[(size_t)y * (W + 1) + x];
        out[(size_t)y * W + x] = (uint32_t)acc;
    }
}

}  // namespace hgs
