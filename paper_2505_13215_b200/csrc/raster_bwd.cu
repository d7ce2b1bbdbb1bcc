// raster_bwd.cu -- K6: tile rasterizer backward (backward.cpp:178-222).
//
// One CTA per tile, re-evaluating every pair with the same arithmetic as K4
// (so every contribute/skip decision is reproduced).  Like the reference it
// walks each pixel's list BACK TO FRONT from the forward's recorded last
// contributor, accumulating the suffix colour already dotted with the pixel
// gradient, GS_i = g . (sum_{j>i} c_j a_j T_j + T_final*bg), by addition
// (accurate for deep, nearly occluded splats, unlike C_out - prefix) and
// recovering T_i = T_{i+1} / (1 - a_i) from the stored final transmittance.
//
// Warp w owns the 8x8 quadrant w of the tile, two pixels (rows y, y+4) per
// lane; splats whose quadrant mask bit is clear are skipped warp-uniformly.
// Per splat and warp the pixels' contributions are summed in registers,
// reduced with a transposing butterfly (14 shuffles instead of 45) and added
// with one red.global.add.f32 instruction per accumulator.  The accumulators
// are conic-free (h = g * dL/da, h*dx, h*dy, h*dx^2, h*dx*dy, h*dy^2): K7
// applies alpha and the FP64 conic once per splat.
// Pixels the forward handed to the FP64 fix-up are back-propagated by
// raster_bwd_exact_kernel (one warp per pixel, FP64).
#include <cstddef>

#include "gauss_math.cuh"
#include "kernels.cuh"
#include "sh.cuh"

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


}  // namespace

// accum layout: kAccStrideHost doubles per sorted splat (16-byte aligned), with
// h = g * dL/da (g = exp(-power), a = alpha * g) and d = pixel - mean:
//   [0..2] sum w * dL/dC (d_rgb), [3] sum h (= d_alpha), [4] sum h dx,
//   [5] sum h dy, [6] sum h dx^2, [7] sum h dx dy, [8] sum h dy^2, [9] pad
// Each warp reduces its pixels in FP32 (at most 64 terms) and adds the warp
// total to the FP64 accumulator (hgs_common.cuh: the FP32 running sum over
// the splat's warps was the dominant gradient error at configs[1]).
// K7 turns [4..8] into d_screen = alpha * conic . ([4],[5]) and
// d_conic = -alpha/2 * ([6] [7]; [7] [8]) (backward.cpp:212-221).
constexpr int kAccStride = kAccStrideHost;
#ifndef HGS_DIRECT_LANES
#define HGS_DIRECT_LANES 8
#endif
constexpr int kDirectLanes = HGS_DIRECT_LANES;  // contributing lanes up to which atomics replace the reduction
constexpr int kThreadsB = 128;  // two pixels per thread

__device__ __forceinline__ void red_add(acc_t* addr, float v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(addr), "d"((double)v) : "memory");
}


__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Reverse-sweep state of a lane's two pixels, packed (lo = row y, hi = row
// y + 4): dL/dC, the transmittance after the current splat, g . suffix colour
// (incl. T_final * bg); last contributor per pixel.
struct PixBwd2 {
    f2 gr, gg, gb;
    f2 T;
    f2 GS;
    uint32_t last0, last1;
};

// One pair of backward.cpp:204-221 for both pixels given the pair alphas
// (p0 / p1 = the pixel's pair contributes): w = a T_i and h = g dL/da (0 when
// the pixel's pair does not contribute), and the state stepped to the front
// of the splat.  Per pixel exactly the scalar sequence
//   a = alpha g; inv = rcp(1 - a); T_i = T inv; gc = g . rgb;
//   dL/da = T_i gc - inv S;  w = a T_i;  h = g dL/da;  S += w gc
__device__ __forceinline__ void backprop_pairs(PixBwd2& s, bool p0, bool p1, f2 G, float alpha_f, const float4 col,
                                               float& w0, float& w1, float& h0, float& h1, f2& W) {
    const f2 A = f2_mul(f2_bc(alpha_f), G);
    const f2 OM = f2_sub(f2_bc(1.0f), A);
    const f2 INV = f2_pk(rcp_approx(f2_lo(OM)), rcp_approx(f2_hi(OM)));
    const f2 TI = f2_mul(s.T, INV);
    const f2 GC = f2_fma(s.gr, f2_bc(col.x), f2_fma(s.gg, f2_bc(col.y), f2_mul(s.gb, f2_bc(col.z))));
    const f2 NS = f2_mul(f2_mul(f2_bc(-1.0f), INV), s.GS);  // (-inv) S, exact negation
    const f2 DA = f2_fma(TI, GC, NS);
    // g (hence a) is exactly 0 for a pixel whose pair does not contribute
    // (exponent 128: ex2.approx.ftz(-128) flushes to +0), so its w and h are
    // 0 and its suffix unchanged without selects; only T needs one (T * rcp(1)
    // is not guaranteed to be T)
    const f2 AT = f2_mul(A, TI);
    const f2 GDA = f2_mul(G, DA);
    w0 = f2_lo(AT);
    w1 = f2_hi(AT);
    h0 = f2_lo(GDA);
    h1 = f2_hi(GDA);
    W = AT;
    s.GS = f2_fma(W, GC, s.GS);
    s.T = f2_pk(p0 ? f2_lo(TI) : f2_lo(s.T), p1 ? f2_hi(TI) : f2_hi(s.T));
}

// FP64 backward of one pixel (backward.cpp:182-221) by one warp over 32-splat
// chunks (exact_chunk).  Pass 0 recomposites the pixel to get C_out (skipped
// when the forward fix-up's FP64 colour `cout` is given); pass 1 walks the
// list again, forms the inclusive colour prefix P_i with a warp scan, and
// every contributing lane emits its gradient with
// d_a = g.(c T_i - (C_out - P_i)/(1 - a)) (in FP64 the subtraction is exact
// enough) via global atomics, in the accumulator layout of raster_bwd_kernel.
// Out of line: K6 calls it for its tile's fix-up pixels after its walk.
static __device__ __noinline__ void exact_bwd_pixel(int pix, uint2 rg, const double* __restrict__ cout,
                                                   const uint32_t* __restrict__ inst_val,
                                                   const SplatRec* __restrict__ exact, int W, double bg_r,
                                                   double bg_g, double bg_b, const uint32_t* __restrict__ last_arr,
                                                   const float* __restrict__ dL_dimg,
                                                   const double* __restrict__ col64, acc_t* __restrict__ accum,
                                                   double* s_om) {
    const int lane = threadIdx.x & 31;
    HGS_DCHECK(pix >= 0 && (unsigned long long)pix < g_chk.pixels);
    const double gp[3] = {dL_dimg[pix * 3], dL_dimg[pix * 3 + 1], dL_dimg[pix * 3 + 2]};
    if (fabs(gp[0]) <= 1e-12 && fabs(gp[1]) <= 1e-12 && fabs(gp[2]) <= 1e-12) return;  // isZero, backward.cpp:189
    const int px = pix % W, py = pix / W;
    const uint32_t last = last_arr[pix] & 0x7fffffffu;
    HGS_DCHECK(rg.x <= rg.y && rg.y <= g_chk.inst && last <= rg.y);
    const double pcx = px + 0.5, pcy = py + 0.5;
    double Cout[3];
    int pass0 = 0;
    if (cout) {
        Cout[0] = cout[0];
        Cout[1] = cout[1];
        Cout[2] = cout[2];
        pass0 = 1;
    }
    for (int pass = pass0; pass < 2; ++pass) {
        double T = 1.0, P[3] = {0.0, 0.0, 0.0};
        constexpr int S = kExactSub;
        for (uint32_t base = rg.x; base < last; base += 32 * S) {
            ExactChunk<S> c;
            exact_chunk<S>(inst_val, exact, nullptr, base, last, px, py, pcx, pcy, T, s_om, c);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                double wc[3] = {0.0, 0.0, 0.0}, w = 0.0, rgb[3] = {0.0, 0.0, 0.0};
                if (c.contrib[s]) {
                    if (col64) {  // exact mode: the FP64 colours
                        const double* cc = col64 + 3 * (size_t)(c.e[s] - exact);
                        rgb[0] = cc[0];
                        rgb[1] = cc[1];
                        rgb[2] = cc[2];
                    } else {
                        rgb[0] = c.e[s]->r;
                        rgb[1] = c.e[s]->g;
                        rgb[2] = c.e[s]->b;
                    }
                    w = __dmul_rn(c.a[s], c.Ti[s]);
                    wc[0] = rgb[0] * w;
                    wc[1] = rgb[1] * w;
                    wc[2] = rgb[2] * w;
                }
                if (pass == 0) {
                    for (int k = 0; k < 3; ++k) P[k] += warp_sum_d(wc[k]);
                    continue;
                }
                // inclusive prefix of this 32-splat slice (list order) on top of the running P
                double inc[3] = {wc[0], wc[1], wc[2]};
#pragma unroll
                for (int o = 1; o < 32; o <<= 1)
                    for (int k = 0; k < 3; ++k) {
                        const double u = __shfl_up_sync(0xffffffffu, inc[k], o);
                        if (lane >= o) inc[k] += u;
                    }
                if (c.contrib[s]) {
                    const SplatRec* e = c.e[s];
                    double d_a = 0.0;
                    for (int k = 0; k < 3; ++k)
                        d_a += gp[k] * (rgb[k] * c.Ti[s] - (Cout[k] - (P[k] + inc[k])) / (1.0 - c.a[s]));
                    acc_t* dst = accum + (size_t)(e - exact) * kAccStride;
                    for (int k = 0; k < 3; ++k) atomicAdd(dst + k, w * gp[k]);
                    const double h = c.g[s] * d_a;
                    const double dx = pcx - e->sx, dy = pcy - e->sy;
                    atomicAdd(dst + 3, h);
                    atomicAdd(dst + 4, h * dx);
                    atomicAdd(dst + 5, h * dy);
                    atomicAdd(dst + 6, h * dx * dx);
                    atomicAdd(dst + 7, h * dx * dy);
                    atomicAdd(dst + 8, h * dy * dy);
                }
                for (int k = 0; k < 3; ++k) P[k] += __shfl_sync(0xffffffffu, inc[k], 31);
            }
            if (c.term >= 0) break;
        }
        if (pass == 0) {
            Cout[0] = P[0] + T * bg_r;
            Cout[1] = P[1] + T * bg_g;
            Cout[2] = P[2] + T * bg_b;
        }
    }
    __syncwarp();
}

// The exact backward mode (hgs_set_exact_backward): every pixel through
// exact_bwd_pixel with the FP64 colours, one warp per pixel.
__global__ void __launch_bounds__(128) raster_bwd_exact_kernel(
    int all_pixels, const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val,
    const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r, double bg_g, double bg_b,
    const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg, const double* __restrict__ col64,
    acc_t* __restrict__ accum) {
    pdl_wait();  // launched with launch_pdl
    __shared__ double s_om[4][32 * kExactSub];
    const int wib = threadIdx.x >> 5;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t q = blockIdx.x * (blockDim.x >> 5) + wib; q < (uint32_t)all_pixels; q += warps) {
        const int pix = (int)q;
        const int px = pix % W, py = pix / W;
        exact_bwd_pixel(pix, ranges[(py / kTile) * tiles_x + px / kTile], nullptr, inst_val, exact, W, bg_r, bg_g,
                        bg_b, last_arr, dL_dimg, col64, accum, s_om[wib]);
    }
}

__global__ void __launch_bounds__(kThreadsB, 8) raster_bwd_kernel(
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val, const SplatFast* __restrict__ fast,
    const SplatRec* __restrict__ exact, int W, int H, int tiles_x, const float* __restrict__ tfinal,
    const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg, float bg_r, float bg_g, float bg_b,
    acc_t* __restrict__ accum, const uint32_t* __restrict__ tile_order, const uint32_t* __restrict__ fix_slot,
    const double* __restrict__ fix_cout, double bg_rd, double bg_gd, double bg_bd) {
    pdl_wait();  // launched with launch_pdl
    __shared__ SplatBatch<kBatchB> sb;
    __shared__ uint32_t s_nfix, s_fix[kThreadsB * 2];  // this tile's fix-up pixels (FP64 backward after the walk)
    __shared__ uint16_t s_list[kThreadsB / 32][kBatchB];  // per-warp splat lists (build_warp_list)
    __shared__ uint32_t s_maxlast;
    const int tile = tile_order ? (int)tile_order[blockIdx.x] : (int)blockIdx.x;  // heaviest tiles first
    const int tx = tile % tiles_x, ty = tile / tiles_x;
    // warp w owns the 8x8 quadrant (w & 1, w >> 1); a lane owns rows y, y+4
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int px = tx * kTile + (warp & 1) * 8 + (lane & 7);
    const int py0 = ty * kTile + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
    HGS_DCHECK((unsigned long long)tile < g_chk.tiles);
    const uint2 rg = ranges[tile];
    HGS_DCHECK(rg.x <= rg.y && rg.y <= g_chk.inst);
    const float pxc = (float)px + 0.5f, pyc0 = (float)py0 + 0.5f, pyc1 = (float)py1 + 0.5f;
    // FP64 pixel centres for the rare exact paths, rebuilt there (opaque: not
    // hoisted into 6 loop-carried registers of the 64)
    auto pcx = [&] { return (double)(int)opaque_u32((uint32_t)px) + 0.5; };
    auto pcy = [&](int py) { return (double)(int)opaque_u32((uint32_t)py) + 0.5; };

    struct Pix1 {
        float gr, gg, gb, T, GS;
        uint32_t last;
    };
    auto init = [&](int py, Pix1& s) {
        s = Pix1{0.f, 0.f, 0.f, 1.f, 0.f, rg.x};
        if (px >= W || py >= H) return;
        const int pix = py * W + px;
        const uint32_t l = last_arr[pix];
        s.gr = dL_dimg[pix * 3 + 0];
        s.gg = dL_dimg[pix * 3 + 1];
        s.gb = dL_dimg[pix * 3 + 2];
        s.T = tfinal[pix];
        s.GS = s.T * fmaf(s.gr, bg_r, fmaf(s.gg, bg_g, s.gb * bg_b));
        // flagged pixels go through the exact kernel; a gradient that is
        // zero by Eigen's isZero (every |component| <= 1e-12, backward.cpp:189;
        // for floats <= 1e-12f is the same test) leaves the pixel untouched
        const bool zero = fabsf(s.gr) <= 1e-12f && fabsf(s.gg) <= 1e-12f && fabsf(s.gb) <= 1e-12f;
        if (!(l & 0x80000000u) && !zero) s.last = l;
        if ((l & 0x80000000u) && !zero) s_fix[atomicAdd(&s_nfix, 1u)] = (uint32_t)pix;
    };
    // the box test's bits in a staged tile-relative mask (column bit | row bit):
    // a pixel is in the box iff both are set
    const int cshift = px - tx * kTile, rshift0 = 16 + py0 - ty * kTile;
    // per-thread loop constants in shared memory (read back with volatile
    // loads where needed): the box-test bits and the FP32 pixel-centre column
    __shared__ uint4 s_pix[kThreadsB];
    s_pix[threadIdx.x] = make_uint4((1u << cshift) | (1u << rshift0), (1u << cshift) | (1u << (rshift0 + 4)),
                                    __float_as_uint(pxc), 0u);
    const uint32_t a_pix = opaque_u32((uint32_t)__cvta_generic_to_shared(&s_pix[threadIdx.x]));
    if (threadIdx.x == 0) s_nfix = 0u;
    __syncthreads();
    PixBwd2 s;
    {
        Pix1 a0, a1;
        init(py0, a0);
        init(py1, a1);
        s.gr = f2_pk(a0.gr, a1.gr);
        s.gg = f2_pk(a0.gg, a1.gg);
        s.gb = f2_pk(a0.gb, a1.gb);
        s.T = f2_pk(a0.T, a1.T);
        s.GS = f2_pk(a0.GS, a1.GS);
        s.last0 = a0.last;
        s.last1 = a1.last;
    }
    const f2 PYC = f2_pk(pyc0, pyc1);
    if (threadIdx.x == 0) s_maxlast = rg.x;
    __syncthreads();
    const uint32_t ml = max(s.last0, s.last1);
    if (ml > rg.x) atomicMax(&s_maxlast, ml);
    __syncthreads();
    const uint32_t end = s_maxlast;
    HGS_DCHECK(end >= rg.x && end <= rg.y);
    const uint32_t warp_end = __reduce_max_sync(0xffffffffu, ml);  // nothing past it in this warp

    using SB = SplatBatch<kBatchB>;
    const uint32_t sbase = opaque_u32((uint32_t)__cvta_generic_to_shared(&sb));
    const uint32_t a_bm = sbase + offsetof(SB, bm), a_hdr = sbase + offsetof(SB, hdr),
                   a_chol = sbase + offsetof(SB, chol), a_col = sbase + offsetof(SB, col),
                   a_mean = sbase + offsetof(SB, mean), a_j = sbase + offsetof(SB, j);
    const int nbatch = (int)((end - rg.x + kBatchB - 1) / kBatchB);
#ifdef HGS_CHECKED
    unsigned long long n_it = 0, n_box = 0, n_pass = 0, n_wit = 0;
#endif
    for (int bi = nbatch - 1; bi >= 0; --bi) {
        const uint32_t base = rg.x + (uint32_t)bi * kBatchB;
        const int nb = (int)min((uint32_t)kBatchB, end - base);
        __syncthreads();
        for (int t = threadIdx.x; t < nb; t += kThreadsB) sb.load(t, fast, inst_val[base + t], tx * kTile, ty * kTile);
        __syncthreads();
        const int kmax = (int)min((uint32_t)nb, warp_end > base ? warp_end - base : 0u);
        if (kmax == 0) continue;  // (warp-uniform; the next batch's barriers are reached by every warp)
        // this warp's splats (quadrant-mask bit set: exact, no pixel of the
        // quadrant reaches 1/255 otherwise), walked back to front below kmax
        const int cnt = build_warp_list<kBatchB>(sb.qm, sb.bm, kmax, warp, s_list[warp]);
        const uint32_t a_list = opaque_u32((uint32_t)__cvta_generic_to_shared(&s_list[warp][0]));
        // splat k of the batch precedes a pixel's last contributor iff
        // 16 k < 16 (last - base) (clamped to [-1, kBatchB]: no overflow)
        const int l0 = max(-1, min((int)kBatchB, (int)s.last0 - (int)base)) * 16;
        const int l1 = max(-1, min((int)kBatchB, (int)s.last1 - (int)base)) * 16;
        for (int q = cnt - 1; q >= 0; --q) {
            const uint32_t le = lds_u16(a_list + 2 * q);
            const uint32_t o16 = le & 0x0ff0u, o4 = o16 >> 2;
            const int4 hdr = lds_i4(a_hdr + o16);
            // box test: known true when the box covers the quadrant, else from
            // the staged tile-relative column/row masks
            bool b0 = (int)o16 < l0, b1 = (int)o16 < l1;
            if (!(le & 0x8000u)) {
                const uint32_t bm = lds_u32(a_bm + o4);
                const uint2 bx = ldsv_u2(a_pix);
                b0 = b0 && (bm & bx.x) == bx.x;
                b1 = b1 && (bm & bx.y) == bx.y;
            }
            if (!__any_sync(0xffffffffu, b0 || b1)) continue;
#ifdef HGS_CHECKED
            ++n_it;
            n_box += (int)b0 + (int)b1;
            if (lane == 0) ++n_wit;
#endif
            const float4 L = lds_f4(a_chol + o16), col = lds_f4(a_col + o16);
            // the splat's index (loaded where used: the rare exact paths and the
            // accumulator address)
            auto sjf = [&] { return lds_u32(a_j + o4); };
            auto rec = [&] { return exact + sjf(); };
            // exponent argument and offset of both pixels (same column: one dx
            // on the fast path, the same rounding sequence as K4's fast_x)
            float x0 = INFINITY, x1 = INFINITY, dx0 = 0.f, dx1 = 0.f, dy0 = 0.f, dy1 = 0.f;
            if (__int_as_float(hdr.w) < 0.0f) {  // FP64 exponent path (uniform per splat)
                if (b0) {
                    x0 = exact_x(rec(), pcx(), pcy(py0));
                    const float2 d = exact_delta(rec(), pcx(), pcy(py0));
                    dx0 = d.x;
                    dy0 = d.y;
                }
                if (b1) {
                    x1 = exact_x(rec(), pcx(), pcy(py1));
                    const float2 d = exact_delta(rec(), pcx(), pcy(py1));
                    dx1 = d.x;
                    dy1 = d.y;
                }
            } else {  // both pixels in one packed sequence (= fast_x per pixel)
                const float4 m = lds_f4(a_mean + o16);
                dx0 = __fsub_rn(__fsub_rn(ldsv_f(a_pix + 8), m.x), m.z);
                dx1 = dx0;
                const f2 DY = f2_sub(f2_sub(PYC, f2_bc(m.y)), f2_bc(m.w));
                const f2 U1 = f2_fma(f2_bc(L.x), f2_bc(dx0), f2_mul(f2_bc(L.y), DY));
                const f2 U2 = f2_mul(f2_bc(L.z), DY);
                const f2 X = f2_fma(U1, U1, f2_mul(U2, U2));
                x0 = f2_lo(X);
                x1 = f2_hi(X);
                dy0 = f2_lo(DY);
                dy1 = f2_hi(DY);
            }
            // the oracle's a >= 1/255 test (exact: FP64 inside the guard band)
            const float x_skip = __int_as_float(hdr.z), x_keep = col.w;
            bool p0 = b0 && x0 < x_skip, p1 = b1 && x1 < x_skip;
            const bool band0 = p0 && x0 >= x_keep, band1 = p1 && x1 >= x_keep;
            if (band0 || band1) {  // rare
                if (band0) p0 = exact_alpha_passes(rec(), pcx(), pcy(py0));
                if (band1) p1 = exact_alpha_passes(rec(), pcx(), pcy(py1));
            }
            // lanes without a contributing pixel hold zeros; skip the
            // reduction when the whole warp is empty
            if (!__any_sync(0xffffffffu, p0 || p1)) continue;
#ifdef HGS_CHECKED
            n_pass += (int)p0 + (int)p1;
#endif
            const float g0 = fast_exp2_neg(p0 ? x0 : 128.0f), g1 = fast_exp2_neg(p1 ? x1 : 128.0f);
            float w0, h0, w1, h1;
            f2 Wp;
            backprop_pairs(s, p0, p1, f2_pk(g0, g1), L.w, col, w0, w1, h0, h1, Wp);
            const float hx0 = h0 * dx0, hx1 = h1 * dx1, hy0 = h0 * dy0, hy1 = h1 * dy1;
            float v[9];
            v[0] = fmaf(w0, f2_lo(s.gr), w1 * f2_hi(s.gr));
            v[1] = fmaf(w0, f2_lo(s.gg), w1 * f2_hi(s.gg));
            v[2] = fmaf(w0, f2_lo(s.gb), w1 * f2_hi(s.gb));
            v[3] = h0 + h1;
            v[4] = hx0 + hx1;
            v[5] = hy0 + hy1;
            v[6] = fmaf(hx0, dx0, hx1 * dx1);
            v[7] = fmaf(hx0, dy0, hx1 * dy1);
            v[8] = fmaf(hy0, dy0, hy1 * dy1);
            const uint32_t sj = sjf();
            HGS_DCHECK(sj < g_chk.splats);
            acc_t* dst = accum + (size_t)sj * kAccStride;
            const unsigned am = __ballot_sync(0xffffffffu, p0 || p1);
            if (__popc(am) <= kDirectLanes) {
                // few contributing lanes: their own atomics are cheaper than the butterfly
                if (p0 || p1)
#pragma unroll
                    for (int q = 0; q < 9; ++q) red_add(dst + q, v[q]);
            } else {
                const float r8 = transpose_reduce8(v);
                const float r9 = warp_sum(v[8]);
                if ((lane & 3) == 0) red_add(dst + (lane >> 2), r8);
                else if (lane == 1) red_add(dst + 8, r9);
            }
        }
    }
#ifdef HGS_CHECKED
    HGS_COUNT_PAIRS(4, n_it);
    HGS_COUNT_PAIRS(5, n_box);
    HGS_COUNT_PAIRS(6, n_pass);
    HGS_COUNT_PAIRS(7, n_wit);
#endif
    // the FP64 backward of this tile's fix-up pixels, one warp per pixel, with
    // the forward fix-up's FP64 colour; the staged batch's memory holds the
    // walks' transmittance factors
    __syncthreads();
    const uint32_t nfix = s_nfix;
    double* s_om = reinterpret_cast<double*>(&sb.mean[0]) + warp * (32 * kExactSub);
    for (uint32_t k = warp; k < nfix; k += kThreadsB / 32) {
        const int pix = (int)s_fix[k];
        exact_bwd_pixel(pix, rg, fix_cout + 3 * (size_t)fix_slot[pix], inst_val, exact, W, bg_rd, bg_gd, bg_bd,
                        last_arr, dL_dimg, nullptr, accum, s_om);
    }
}

// ---- exact backward mode (hgs_set_exact_backward): FP64 colours of the
// visible splats for the FP64 pixel walk.
// FP64 colour of a Gaussian (sh.cpp:73-83; view direction raster.cpp:83-85
// from the conditional mean, gauss_math.cpp:175-186).
__device__ void exact_colour(int gid, int n4, const float* __restrict__ p4, int64_t cap4,
                             const float* __restrict__ p3, int64_t cap3, int deg, const DevCamera& cam, double t,
                             double out[3]) {
    double mean3[3];
    const float* P;
    int64_t cap;
    int i, shrow;
    if (gid < n4) {
        i = gid;
        P = p4;
        cap = cap4;
        shrow = R4_SH;
        double ql[4], qr[4], es[4];
        for (int k = 0; k < 4; ++k) {
            ql[k] = p4[(int64_t)(R4_QL + k) * cap4 + i];
            qr[k] = p4[(int64_t)(R4_QR + k) * cap4 + i];
            es[k] = exp((double)p4[(int64_t)(R4_LS + k) * cap4 + i]);
        }
        const gm::M4 R = gm::rot4_from_pair(ql, qr);
        double cov[4];  // column 3 of R diag(e^s)^2 R^T
        for (int a = 0; a < 4; ++a) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s += (R.a[a][k] * es[k]) * (R.a[3][k] * es[k]);
            cov[a] = s;
        }
        const double dt = t - (double)p4[(int64_t)R4_MT * cap4 + i];
        for (int k = 0; k < 3; ++k) mean3[k] = (double)p4[(int64_t)(R4_MEAN + k) * cap4 + i] + cov[k] * (dt / cov[3]);
    } else {
        i = gid - n4;
        P = p3;
        cap = cap3;
        shrow = R3_SH;
        for (int k = 0; k < 3; ++k) mean3[k] = p3[(int64_t)(R3_MEAN + k) * cap3 + i];
    }
    const double v[3] = {mean3[0] - cam.pos[0], mean3[1] - cam.pos[1], mean3[2] - cam.pos[2]};
    const double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    double d[3] = {0.0, 0.0, 1.0};
    if (nrm > 0.0)
        for (int k = 0; k < 3; ++k) d[k] = v[k] / nrm;
    double basis[16];
    sh_basis_t<double>(d, deg, basis);
    const int K = sh_count(deg);
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) acc += (double)P[(int64_t)(shrow + 3 * k + c) * cap + i] * basis[k];
        out[c] = fmin(fmax(acc + 0.5, 0.0), 1.0);
    }
}

__global__ void __launch_bounds__(128) exact_colour_kernel(const uint32_t* __restrict__ sorted_gid, int V, int n4,
                                                           const float* __restrict__ p4, int64_t cap4,
                                                           const float* __restrict__ p3, int64_t cap3, int deg,
                                                           DevCamera cam, double t, double* __restrict__ col64) {
    pdl_wait();  // launched with launch_pdl
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < V) exact_colour((int)sorted_gid[j], n4, p4, cap4, p3, cap3, deg, cam, t, col64 + 3 * (size_t)j);
}

}  // namespace hgs
