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
#include "hgs_common.cuh"
#include "raster_common.cuh"
#include "sh.cuh"
#include "gauss_math.cuh"

namespace hgs {

namespace {

using gm::M3;
using gm::M4;
using gm::rot4_from_pair;
using gm::quat_to_rot3;

// gauss_math.cpp:159-162
__device__ inline M4 build_cov4(const M4& rot, const double ls[4]) {
    double e[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) e[j] = exp(ls[j]);
    double m[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) m[i][j] = rot.a[i][j] * e[j];
    M4 r;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            double s = m[i][0] * m[j][0];
            s = s + m[i][1] * m[j][1];
            s = s + m[i][2] * m[j][2];
            s = s + m[i][3] * m[j][3];
            r.a[i][j] = s;
        }
    return r;
}

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
    const double sx = cam.fx * p[0] / z + cam.cx;
    const double sy = cam.fy * p[1] / z + cam.cy;
    double J[2][3];
    J[0][0] = cam.fx / z;
    J[0][1] = 0.0;
    J[0][2] = -cam.fx * p[0] / (z * z);
    J[1][0] = 0.0;
    J[1][1] = cam.fy / z;
    J[1][2] = -cam.fy * p[1] / (z * z);
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
    s.c00 = c2[1][1] / det;
    s.c01 = -c2[0][1] / det;
    s.c10 = -c2[1][0] / det;
    s.c11 = c2[0][0] / det;
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

// K1.  stats[0..5] = culled_depth, culled_offscreen, culled_degenerate,
// culled_temporal, degenerate_temporal, projected.
__global__ void __launch_bounds__(256, 3) preprocess_kernel(
    const float* __restrict__ p4, int64_t cap4, int n4, const float* __restrict__ p3, int64_t cap3,
    int n3, int deg, DevCamera cam, double t, double cutoff, int tiles_x, SplatRec* __restrict__ rec,
    uint32_t* __restrict__ depth_key, uint32_t* __restrict__ ntiles_out,
    unsigned long long* __restrict__ stats, uint32_t* __restrict__ flags, ShRec* __restrict__ shrec) {
    pdl_wait();  // launched with launch_pdl
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = n4 + n3;
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
                ql[k] = __ldg(&p4[(int64_t)(R4_QL + k) * cap4 + i]);
                qr[k] = __ldg(&p4[(int64_t)(R4_QR + k) * cap4 + i]);
                ls[k] = __ldg(&p4[(int64_t)(R4_LS + k) * cap4 + i]);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) mean4[k] = __ldg(&p4[(int64_t)(R4_MEAN + k) * cap4 + i]);
            mean4[3] = __ldg(&p4[(int64_t)R4_MT * cap4 + i]);
            const M4 cov4 = build_cov4(rot4_from_pair(ql, qr), ls);
            // condition_at_time (gauss_math.cpp:175-186)
            const double s44 = cov4.a[3][3];
            if (s44 < 1e-12) {
                reason = CULL_DEGEN_TEMPORAL;
            } else {
                const double cross[3] = {cov4.a[0][3], cov4.a[1][3], cov4.a[2][3]};
                const double dt = t - mean4[3];
                const double f = dt / s44;
#pragma unroll
                for (int k = 0; k < 3; ++k) mean3[k] = mean4[k] + cross[k] * f;
                M3 c;
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) c.a[a][b] = cov4.a[a][b] - (cross[a] * cross[b]) / s44;
                // clamp_psd: lambda_min(Schur complement) >= lambda_min(cov4) = exp(2 min s);
                // the eigen-solve can only change the result when that bound is near 1e-12.
                double smin = fmin(fmin(ls[0], ls[1]), fmin(ls[2], ls[3]));
                double smax = fmax(fmax(ls[0], ls[1]), fmax(ls[2], ls[3]));
                double lam_lo = exp(2.0 * smin), scale = exp(2.0 * smax);
                if (!(lam_lo - 1e-13 * scale >= 1e-12)) ok = clamp_psd_slow(c);
                if (!ok) flag |= FLAG_INDEFINITE;
                const double w = exp(-0.5 * dt * dt / s44);
                if (w < cutoff) {
                    reason = CULL_TEMPORAL;
                } else {
                    reason = project_3d(mean3, c, cam, s, depth, ntiles, tiles_x);
                    if (reason == CULL_NONE)
                        alpha = fmin(sigmoid((double)__ldg(&p4[(int64_t)R4_OP * cap4 + i])) * w, kAlphaClamp);
                }
            }
        } else {
            const int i = gid - n4;
            double q[4], ls[3];
#pragma unroll
            for (int k = 0; k < 4; ++k) q[k] = __ldg(&p3[(int64_t)(R3_Q + k) * cap3 + i]);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                ls[k] = __ldg(&p3[(int64_t)(R3_LS + k) * cap3 + i]);
                mean3[k] = __ldg(&p3[(int64_t)(R3_MEAN + k) * cap3 + i]);
            }
            M3 rot;
            if (!quat_to_rot3(q, rot)) flag |= FLAG_NONUNIT_QUAT;
            const M3 cov3 = build_cov3(rot, ls);
            reason = project_3d(mean3, cov3, cam, s, depth, ntiles, tiles_x);
            if (reason == CULL_NONE)
                alpha = fmin(sigmoid((double)__ldg(&p3[(int64_t)R3_OP * cap3 + i])), kAlphaClamp);
        }
        if (reason == CULL_NONE) {
            // view direction (raster.cpp:83-85) and SH colour
            double v[3] = {mean3[0] - cam.pos[0], mean3[1] - cam.pos[1], mean3[2] - cam.pos[2]};
            double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            double d[3] = {0.0, 0.0, 1.0};
            if (nrm > 0.0) {
                d[0] = v[0] / nrm;
                d[1] = v[1] / nrm;
                d[2] = v[2] / nrm;
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
            float basis[16];
            sh_basis_f(fd, deg, basis);
            ShRec sr;
            float* jr[3] = {&sr.j[0].x, &sr.j[1].x, &sr.j[2].x};
            uint32_t clamped = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                float w[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) w[k] = k < K ? __ldg(&P[(int64_t)(shrow + 3 * k + c) * cap + i]) : 0.f;
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (k < K) acc = fmaf(basis[k], w[k], acc);
                const float raw = acc + 0.5f;  // raster.cpp:86 / sh.cpp:81
                clamped |= (raw < 0.0f || raw > 1.0f) ? (1u << c) : 0u;
                rgb[c] = fminf(fmaxf(raw, 0.0f), 1.0f);
                float g[3];
                sh_dir_grad_f(fd, deg, w, g);
                jr[c][0] = g[0];
                jr[c][1] = g[1];
                jr[c][2] = g[2];
                jr[c][3] = 0.f;
            }
            sr.dir = make_float4(fd[0], fd[1], fd[2], __uint_as_float(clamped));
            shrec[gid] = sr;
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
    // warp-aggregated RenderStats counters
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < kNumStats; ++k) {
        const uint32_t want = k == 0 ? CULL_DEPTH : k == 1 ? CULL_OFFSCREEN : k == 2 ? CULL_DEGENERATE
                             : k == 3 ? CULL_TEMPORAL : k == 4 ? CULL_DEGEN_TEMPORAL : CULL_NONE;
        const unsigned b = __ballot_sync(full, reason == want);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&stats[k], (unsigned long long)__popc(b));
    }
    const unsigned fb = __reduce_or_sync(full, flag);
    if ((threadIdx.x & 31) == 0 && fb) atomicOr(flags, fb);
}

}  // namespace hgs
