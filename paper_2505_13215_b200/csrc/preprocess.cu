// preprocess.cu -- K1: fused 4D->3D conditional slice + EWA projection + SH.
//
// One thread per Gaussian (4D pool first, then 3D: gid = i / n4 + i), the
// reference's project_scene order (raster.cpp:90-116).  Geometry is FP64 and
// this translation unit is compiled with -fmad=false, so every product/sum
// below rounds exactly like the oracle's -ffp-contract=off code: the depth
// f32 bits, the pixel box and therefore the tile assignment and sort keys are
// bit-identical to the CPU reference path.  SH colour is FP32 (it only feeds
// the toleranced image).
//
// Reads 68 B (4D) / 44 B (3D) of geometry + 4*3K B of SH per Gaussian, all
// coalesced from the component-major SoA pools; writes an 80 B SplatRec, a
// depth key and a tile count.  Bound: HBM.
#include <atomic>
#include "hgs_common.cuh"
#include "raster_common.cuh"
#include "sh.cuh"
#include "gauss_math.cuh"
#include "tma.cuh"

namespace hgs {

namespace {

using gm::M3;
using gm::M4;
using gm::rot4_from_pair;
using gm::quat_to_rot3;

// gauss_math.cpp:154-157
__device__ inline M3 build_cov3(const M3& rot, const double ls[3]) {
    double e[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double m[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) m[i][j] = rot.a[i][j] * e[j];
    M3 r;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double s = m[i][0] * m[j][0];
            s = s + m[i][1] * m[j][1];
            s = s + m[i][2] * m[j][2];
            r.a[i][j] = s;
        }
    return r;
}

// Cyclic Jacobi for the rare clamp_psd eigen path (gauss_math.cpp:164-173);
// same algorithm and operation order as the oracle's jacobi_eig3.
__device__ __noinline__ void jacobi_eig3(const M3& in, double ev[3], M3& v) {
    M3 a = in;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v.a[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = fabs(a.a[0][1]) + fabs(a.a[0][2]) + fabs(a.a[1][2]);
        double diag = fabs(a.a[0][0]) + fabs(a.a[1][1]) + fabs(a.a[2][2]);
        if (off <= 1e-300 || off <= 1e-18 * diag) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = a.a[p][q];
                if (apq == 0.0) continue;
                double theta = (a.a[q][q] - a.a[p][p]) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {
                    double akp = a.a[k][p], akq = a.a[k][q];
                    a.a[k][p] = c * akp - s * akq;
                    a.a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    double apk = a.a[p][k], aqk = a.a[q][k];
                    a.a[p][k] = c * apk - s * aqk;
                    a.a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    double vkp = v.a[k][p], vkq = v.a[k][q];
                    v.a[k][p] = c * vkp - s * vkq;
                    v.a[k][q] = s * vkp + c * vkq;
                }
            }
    }
    int idx[3] = {0, 1, 2};
    // insertion sort ascending by eigenvalue (std::sort on 3 keys in the oracle)
    for (int i = 1; i < 3; ++i)
        for (int j = i; j > 0 && a.a[idx[j]][idx[j]] < a.a[idx[j - 1]][idx[j - 1]]; --j) {
            int tmp = idx[j];
            idx[j] = idx[j - 1];
            idx[j - 1] = tmp;
        }
    M3 vs;
    for (int c = 0; c < 3; ++c) {
        ev[c] = a.a[idx[c]][idx[c]];
        for (int r = 0; r < 3; ++r) vs.a[r][c] = v.a[r][idx[c]];
    }
    v = vs;
}

// clamp_psd's slow path: returns false if the matrix is indefinite.
__device__ __noinline__ bool clamp_psd_slow(M3& m) {
    M3 sym;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sym.a[i][j] = 0.5 * (m.a[i][j] + m.a[j][i]);
    double ev[3];
    M3 v;
    jacobi_eig3(sym, ev, v);
    double min_ev = fmin(ev[0], fmin(ev[1], ev[2]));
    if (min_ev >= 1e-12) {
        m = sym;
        return true;
    }
    if (min_ev < -1e-8) return false;
    M3 vd;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) vd.a[i][j] = v.a[i][j] * fmax(ev[j], 1e-12);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = vd.a[i][0] * v.a[j][0];
            s = s + vd.a[i][1] * v.a[j][1];
            s = s + vd.a[i][2] * v.a[j][2];
            m.a[i][j] = s;
        }
    return true;
}

__device__ inline uint32_t f32_bits(double d) { return __float_as_uint(__double2float_rn(d)); }

// project_3d (raster.cpp:26-64).  Returns the cull reason (CULL_NONE when
// projected) and fills the geometric part of the record.
__device__ inline uint32_t project_3d(const double m[3], const M3& cov, const DevCamera& cam, SplatRec& s,
                                      double& depth, int& ntiles, int tiles_x) {
    double p[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        double a = cam.R[i * 3 + 0] * m[0];
        a = a + cam.R[i * 3 + 1] * m[1];
        a = a + cam.R[i * 3 + 2] * m[2];
        p[i] = a + cam.t[i];
    }
    const double z = p[2];
    if (z < cam.near_ || z > cam.far_) return CULL_DEPTH;
    depth = z;
    // the six divisions by z and z*z through two reciprocals (gm::Rcp: bit-identical quotients)
    const gm::Rcp rz(z), rzz(z * z);
    const double sx = rz.div(cam.fx * p[0]) + cam.cx;
    const double sy = rz.div(cam.fy * p[1]) + cam.cy;
    double J[2][3];
    J[0][0] = rz.div(cam.fx);
    J[0][1] = 0.0;
    J[0][2] = rzz.div(-cam.fx * p[0]);
    J[1][0] = 0.0;
    J[1][1] = rz.div(cam.fy);
    J[1][2] = rzz.div(-cam.fy * p[1]);
    double T[2][3];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double a = J[i][0] * cam.R[0 * 3 + k];
            a = a + J[i][1] * cam.R[1 * 3 + k];
            a = a + J[i][2] * cam.R[2 * 3 + k];
            T[i][k] = a;
        }
    double tc[2][3];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            double a = T[i][0] * cov.a[0][k];
            a = a + T[i][1] * cov.a[1][k];
            a = a + T[i][2] * cov.a[2][k];
            tc[i][k] = a;
        }
    double c2[2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            double a = tc[i][0] * T[j][0];
            a = a + tc[i][1] * T[j][1];
            a = a + tc[i][2] * T[j][2];
            c2[i][j] = a;
        }
    c2[0][0] += kLowPass;
    c2[1][1] += kLowPass;
    const double det = c2[0][0] * c2[1][1] - c2[0][1] * c2[1][0];
    if (det <= 1e-12) return CULL_DEGENERATE;
    const gm::Rcp rdet(det);
    s.c00 = rdet.div(c2[1][1]);
    s.c01 = rdet.div(-c2[0][1]);
    s.c10 = rdet.div(-c2[1][0]);
    s.c11 = rdet.div(c2[0][0]);
    const double mid = 0.5 * (c2[0][0] + c2[1][1]);
    const double max_ev = mid + sqrt(fmax(0.0, mid * mid - det));
    const int radius = (int)ceil(3.0 * sqrt(max_ev));
    const int mx = (int)floor(sx), my = (int)floor(sy);
    const int x0 = max(0, mx - radius), x1 = min(cam.width - 1, mx + radius);
    const int y0 = max(0, my - radius), y1 = min(cam.height - 1, my + radius);
    if (x0 > x1 || y0 > y1) return CULL_OFFSCREEN;
    s.sx = sx;
    s.sy = sy;
    s.x0 = (int16_t)x0;
    s.x1 = (int16_t)x1;
    s.y0 = (int16_t)y0;
    s.y1 = (int16_t)y1;
    ntiles = (x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1);
    (void)tiles_x;
    return CULL_NONE;
}

__device__ inline double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

}  // namespace

// Shared-memory staging of a block's parameter columns: one 1D bulk copy
// (TMA) per parameter row of the block's 256 Gaussians, all issued at block
// start by one thread and completed on an mbarrier, so the block's whole
// 17-65 row working set is in flight at once (the per-thread loads of the
// FP64 slice and of the 48 SH rows used to be exposed one latency after the
// other).  Row stride 260 floats: the 3D pool's columns start at any
// Gaussian index, so a row is copied from the 16-byte-aligned index below
// and read at offset (0..3).
constexpr int kPreThreads = 256;
constexpr int kPreStride = kPreThreads + 4;
size_t preprocess_smem_bytes(int deg) { return (size_t)rows4(deg) * kPreStride * sizeof(float); }
__global__ void preprocess_kernel(const float* __restrict__ p4, int64_t cap4, int n4, const float* __restrict__ p3,
                                  int64_t cap3, int n3, int deg, DevCamera cam, double t, double cutoff, int tiles_x,
                                  SplatRec* __restrict__ rec, uint32_t* __restrict__ depth_key,
                                  uint32_t* __restrict__ ntiles_out, unsigned long long* __restrict__ stats,
                                  uint32_t* __restrict__ flags, ShRec* __restrict__ shrec);
__global__ void preprocess_render_kernel(const float* __restrict__ p4, int64_t cap4, int n4,
                                         const float* __restrict__ p3, int64_t cap3, int n3, int deg, DevCamera cam,
                                         double t, double cutoff, int tiles_x, SplatRec* __restrict__ rec,
                                         uint32_t* __restrict__ depth_key, uint32_t* __restrict__ ntiles_out,
                                         unsigned long long* __restrict__ stats, uint32_t* __restrict__ flags,
                                         ShRec* __restrict__ shrec);
cudaError_t preprocess_setup() {  // the attribute is per device: set it once on each
    static std::atomic<unsigned long long> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load() & bit) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(preprocess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)preprocess_smem_bytes(3));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(preprocess_render_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)preprocess_smem_bytes(3));
    if (e == cudaSuccess) done.fetch_or(bit);
    return e;
}

// K1.  stats[0..5] = culled_depth, culled_offscreen, culled_degenerate,
// culled_temporal, degenerate_temporal, projected.  kTape: also the SH
// colour's direction Jacobian and clamp mask for the backward (ShRec);
// render sweep frames whose tape is not kept skip them.
template <bool kTape>
__device__ __forceinline__ void preprocess_body(
    const float* __restrict__ p4, int64_t cap4, int n4, const float* __restrict__ p3, int64_t cap3,
    int n3, int deg, DevCamera cam, double t, double cutoff, int tiles_x, SplatRec* __restrict__ rec,
    uint32_t* __restrict__ depth_key, uint32_t* __restrict__ ntiles_out,
    unsigned long long* __restrict__ stats, uint32_t* __restrict__ flags, ShRec* __restrict__ shrec) {
    pdl_wait();  // launched with launch_pdl
    extern __shared__ __align__(128) float s_cols[];  // [row][kPreStride]
    // two transaction barriers: the geometry rows, then the SH rows (the FP64
    // geometry runs while the SH rows are still in flight)
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ uint32_t s_stat[kNumStats], s_done;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = n4 + n3;
    // the block's rows: one pool only (a block straddling the 4D/3D boundary
    // reads global memory directly)
    const int g0 = blockIdx.x * kPreThreads, g1 = min(g0 + kPreThreads, n);
    const bool staged = g1 <= n4 || g0 >= n4;
    const bool sdyn = g1 <= n4;
    const int si0 = sdyn ? g0 : g0 - n4;
    const int soff = staged ? si0 - (si0 & ~3) : 0;  // 16-byte aligned copy start
    if (threadIdx.x < kNumStats) s_stat[threadIdx.x] = 0u;
    if (threadIdx.x == 0) {
        s_done = 0u;
        if (staged) {
            mbar_init(&s_bar[0], 1);
            mbar_init(&s_bar[1], 1);
            const int ngeo = sdyn ? R4_SH : R3_SH, nrows = sdyn ? rows4(deg) : rows3(deg);
            const uint32_t bytes = (uint32_t)(((g1 - g0 + soff + 3) & ~3) * sizeof(float));
            mbar_arrive_expect_tx(&s_bar[0], bytes * (uint32_t)ngeo);
            mbar_arrive_expect_tx(&s_bar[1], bytes * (uint32_t)(nrows - ngeo));
            const float* src = (sdyn ? p4 : p3) + (si0 - soff);
            const int64_t cap = sdyn ? cap4 : cap3;
            for (int r = 0; r < nrows; ++r)
                bulk_g2s(s_cols + r * kPreStride, src + r * cap, bytes, &s_bar[r < ngeo ? 0 : 1]);
        }
    }
    __syncthreads();  // statistics zeroed, barriers initialised
    if (staged) mbar_wait_parity(&s_bar[0], 0);
    // parameter row `row` of this thread's Gaussian (pool P, index i)
    auto ld = [&](const float* __restrict__ P, int64_t cap, int row, int i) -> float {
        return staged ? s_cols[row * kPreStride + soff + (int)threadIdx.x] : __ldg(&P[(int64_t)row * cap + i]);
    };
    uint32_t reason = CULL_DEPTH + 100;  // sentinel: inactive lane
    uint32_t flag = 0;
    if (gid < n) {
        SplatRec s;
        double mean3[3];
        double depth = 0.0;
        int ntiles = 0;
        double alpha = 0.0;
        bool ok = true;
        if (gid < n4) {
            const int i = gid;
            double ql[4], qr[4], ls[4], mean4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                ql[k] = ld(p4, cap4, R4_QL + k, i);
                qr[k] = ld(p4, cap4, R4_QR + k, i);
                ls[k] = ld(p4, cap4, R4_LS + k, i);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) mean4[k] = ld(p4, cap4, R4_MEAN + k, i);
            mean4[3] = ld(p4, cap4, R4_MT, i);
            // cov4 = M M^T with M = rot4 diag(exp(s)) (gauss_math.cpp:159-162);
            // its entries are formed on demand below with build_cov4's
            // operation order (entry (i, j) and (j, i) round identically)
            const M4 rot = rot4_from_pair(ql, qr);
            double e4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) e4[j] = exp(ls[j]);
            double m[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int j = 0; j < 4; ++j) m[a][j] = rot.a[a][j] * e4[j];
            auto cov4 = [&](int a, int b) {
                double sum = m[a][0] * m[b][0];
                sum = sum + m[a][1] * m[b][1];
                sum = sum + m[a][2] * m[b][2];
                sum = sum + m[a][3] * m[b][3];
                return sum;
            };
            // condition_at_time (gauss_math.cpp:175-186)
            const double s44 = cov4(3, 3);
            if (s44 < 1e-12) {
                reason = CULL_DEGEN_TEMPORAL;
            } else {
                const double dt = t - mean4[3];
                const gm::Rcp r44(s44);  // the 11 divisions by s44 through one reciprocal
                const double w = exp(r44.div(-0.5 * dt * dt));
                // clamp_psd: lambda_min(Schur complement) >= lambda_min(cov4) = exp(2 min s);
                // the eigen-solve can only change the result when that bound is near 1e-12.
                // Sufficient without exp: 2 smin >= -27 and 2 (smax - smin) <= 27 give
                // lam_lo - 1e-13 scale >= (1 - 0.054) e^-27 > 1e-12.
                const double smin = fmin(fmin(ls[0], ls[1]), fmin(ls[2], ls[3]));
                const double smax = fmax(fmax(ls[0], ls[1]), fmax(ls[2], ls[3]));
                bool psd_fast = 2.0 * smin >= -27.0 && 2.0 * (smax - smin) <= 27.0;
                if (!psd_fast) psd_fast = exp(2.0 * smin) - 1e-13 * exp(2.0 * smax) >= 1e-12;
                if (w < cutoff && psd_fast) {
                    // temporally culled, and clamp_psd provably neither throws nor
                    // changes anything: the slice itself is never needed
                    reason = CULL_TEMPORAL;
                } else {
                const double cross[3] = {cov4(0, 3), cov4(1, 3), cov4(2, 3)};
                const double f = r44.div(dt);
#pragma unroll
                for (int k = 0; k < 3; ++k) mean3[k] = mean4[k] + cross[k] * f;
                M3 c;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = a; b < 3; ++b) {
                        c.a[a][b] = cov4(a, b) - r44.div(cross[a] * cross[b]);
                        c.a[b][a] = c.a[a][b];
                    }
                if (!psd_fast) {  // (a copy: c's address must not escape the hot path,
                    M3 m = c;      // or it lives in local memory for every Gaussian)
                    ok = clamp_psd_slow(m);
                    c = m;
                }
                if (!ok) flag |= FLAG_INDEFINITE;
                if (w < cutoff) {
                    reason = CULL_TEMPORAL;
                } else {
                    reason = project_3d(mean3, c, cam, s, depth, ntiles, tiles_x);
                    if (reason == CULL_NONE)
                        alpha = fmin(sigmoid((double)ld(p4, cap4, R4_OP, i)) * w, kAlphaClamp);
                }
                }
            }
        } else {
            const int i = gid - n4;
            double q[4], ls[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = ld(p3, cap3, R3_Q + k, i);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                ls[k] = ld(p3, cap3, R3_LS + k, i);
                mean3[k] = ld(p3, cap3, R3_MEAN + k, i);
            }
            M3 rot;
            if (!quat_to_rot3(q, rot)) flag |= FLAG_NONUNIT_QUAT;
            const M3 cov3 = build_cov3(rot, ls);
            reason = project_3d(mean3, cov3, cam, s, depth, ntiles, tiles_x);
            if (reason == CULL_NONE)
                alpha = fmin(sigmoid((double)ld(p3, cap3, R3_OP, i)), kAlphaClamp);
        }
        if (reason == CULL_NONE) {
            // view direction (raster.cpp:83-85) and SH colour
            double v[3] = {mean3[0] - cam.pos[0], mean3[1] - cam.pos[1], mean3[2] - cam.pos[2]};
            double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            double d[3] = {0.0, 0.0, 1.0};
            if (nrm > 0.0) {
                const gm::Rcp rn(nrm);
                d[0] = rn.div(v[0]);
                d[1] = rn.div(v[1]);
                d[2] = rn.div(v[2]);
            }
            // SH colour (sh.cpp:73-83, FP32) and, for the SH backward (K7b: it
            // then needs no SH coefficient), the view direction, the
            // clamped-channel mask and d rgb / d direction -- one channel at a
            // time, each coefficient loaded once
            float rgb[3];
            const float fd[3] = {(float)d[0], (float)d[1], (float)d[2]};
            const float* P = gid < n4 ? p4 : p3;
            const int64_t cap = gid < n4 ? cap4 : cap3;
            const int i = gid < n4 ? gid : gid - n4;
            const int shrow = gid < n4 ? R4_SH : R3_SH;
            const int K = sh_count(deg);
            if (staged) mbar_wait_parity(&s_bar[1], 0);  // the SH rows
            float basis[16];
            sh_basis_f(fd, deg, basis);
            // coefficient-major: the 3 channel values of 4 coefficients in flight
            // at a time, each folded into the 3 colour sums (the same per-channel
            // FMA order as sh.cpp:78-80) and, through the direction factors of
            // that coefficient (dY_k / d(dir), explicit FMAs), into the Jacobian
            float acc[3] = {0.f, 0.f, 0.f}, jg[3][3] = {{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
            const float x = fd[0], y = fd[1], z = fd[2];
#pragma unroll
            for (int k0 = 0; k0 < 16; k0 += 4) {
                float w[4][3];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        w[kk][c] = k0 + kk < K ? ld(P, cap, shrow + 3 * (k0 + kk) + c, i) : 0.f;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int k = k0 + kk;
                    if (k >= K) continue;
                    float f[3] = {0.f, 0.f, 0.f};
                    if (kTape) sh_dir_factor(k, x, y, z, f);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        acc[c] = fmaf(basis[k], w[kk][c], acc[c]);
#pragma unroll
                        for (int j = 0; j < 3; ++j)
                            if (kTape && sh_dir_nonzero(k, j)) jg[c][j] = __fmaf_rn(f[j], w[kk][c], jg[c][j]);
                    }
                }
            }
            ShRec sr;
            uint32_t clamped = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const float raw = acc[c] + 0.5f;  // raster.cpp:86 / sh.cpp:81
                clamped |= (raw < 0.0f || raw > 1.0f) ? (1u << c) : 0u;
                rgb[c] = fminf(fmaxf(raw, 0.0f), 1.0f);
                sr.j[c] = make_float4(jg[c][0], jg[c][1], jg[c][2], 0.f);
            }
            sr.dir = make_float4(fd[0], fd[1], fd[2], __uint_as_float(clamped));
            if (kTape) shrec[gid] = sr;
            s.alpha = alpha;
            s.alpha_f = (float)alpha;
            s.r = rgb[0];
            s.g = rgb[1];
            s.b = rgb[2];
            rec[gid] = s;
            depth_key[gid] = f32_bits(depth);
            ntiles_out[gid] = (uint32_t)ntiles;
        } else {
            ntiles_out[gid] = 0u;
        }
    }
    // RenderStats counters: warp ballots -> block totals in shared memory ->
    // one global atomic per statistic and block, on the block's stripe
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < kNumStats; ++k) {
        const uint32_t want = k == 0 ? CULL_DEPTH : k == 1 ? CULL_OFFSCREEN : k == 2 ? CULL_DEGENERATE
                             : k == 3 ? CULL_TEMPORAL : k == 4 ? CULL_DEGEN_TEMPORAL : CULL_NONE;
        const unsigned b = __ballot_sync(full, reason == want);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&s_stat[k], (uint32_t)__popc(b));
    }
    // the block's last warp to get here flushes the totals (no block barrier:
    // warps of culled Gaussians leave early instead of waiting for the rest)
    uint32_t last = 0;
    if ((threadIdx.x & 31) == 0) {
        __threadfence_block();
        last = atomicAdd(&s_done, 1u) == blockDim.x / 32 - 1 ? 1u : 0u;
    }
    if (__shfl_sync(full, last, 0)) {
        __threadfence_block();
        const int lane = threadIdx.x & 31;
        if (lane < kNumStats) {
            const uint32_t v = atomicAdd(&s_stat[lane], 0u);  // (an atomic read: ordered after the others)
            if (v) atomicAdd(&stats[(blockIdx.x % kStatStripes) * kStatStride + lane], (unsigned long long)v);
        }
    }
    const unsigned fb = __reduce_or_sync(full, flag);
    if ((threadIdx.x & 31) == 0 && fb) atomicOr(flags, fb);
}

#define HGS_K1_PARAMS                                                                                         \
    const float *__restrict__ p4, int64_t cap4, int n4, const float *__restrict__ p3, int64_t cap3, int n3, \
        int deg, DevCamera cam, double t, double cutoff, int tiles_x, SplatRec *__restrict__ rec,           \
        uint32_t *__restrict__ depth_key, uint32_t *__restrict__ ntiles_out,                                \
        unsigned long long *__restrict__ stats, uint32_t *__restrict__ flags, ShRec *__restrict__ shrec
#define HGS_K1_ARGS p4, cap4, n4, p3, cap3, n3, deg, cam, t, cutoff, tiles_x, rec, depth_key, ntiles_out, stats, flags, shrec

__global__ void __launch_bounds__(kPreThreads, 3) preprocess_kernel(HGS_K1_PARAMS) {
    preprocess_body<true>(HGS_K1_ARGS);
}
// render-only (sweep frames without a kept tape; density maps): no ShRec
__global__ void __launch_bounds__(kPreThreads, 3) preprocess_render_kernel(HGS_K1_PARAMS) {
    preprocess_body<false>(HGS_K1_ARGS);
}

}  // namespace hgs
