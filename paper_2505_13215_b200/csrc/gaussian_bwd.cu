// gaussian_bwd.cu -- K7: per-Gaussian backward (backward.cpp:224-354).
//
// One thread per visible (depth-sorted) splat.  Reads the 9 compositing
// accumulators of K6, re-derives the forward intermediates of its Gaussian in
// FP64 from the FP32 parameters (slice, projection Jacobian, view direction,
// raw SH colour) and chains conic -> 2D covariance -> 3D covariance / camera
// mean -> parameters.  4D Gaussians additionally go through the Schur
// complement backward and the isoclinic rotation factors.  Writes
// grad += scale * d, the per-image screen-space norm, and the densification
// statistics (train.cpp:433-444).  Coalesced SoA reads/writes; HBM bound.
#include "kernels.cuh"
#include "sh.cuh"

namespace hgs {

namespace {

__device__ inline void isoL(const double q[4], double L[4][4]) {
    const double a = q[0], b = q[1], c = q[2], d = q[3];
    const double m[4][4] = {{a, -b, -c, -d}, {b, a, -d, c}, {c, d, a, -b}, {d, -c, b, a}};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) L[i][j] = m[i][j];
}
__device__ inline void isoR(const double q[4], double R[4][4]) {
    const double p = q[0], x = q[1], r = q[2], s = q[3];
    const double m[4][4] = {{p, -x, -r, -s}, {x, p, s, -r}, {r, -s, p, x}, {s, r, -x, p}};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) R[i][j] = m[i][j];
}

__device__ inline double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }


}  // namespace

__global__ void __launch_bounds__(128, 4) gaussian_bwd_kernel(
    int N, const uint32_t* __restrict__ sorted_of_gid, const float* __restrict__ accum, int acc_stride, int n4,
    const float* __restrict__ p4, int64_t cap4, const float* __restrict__ p3, int64_t cap3, int deg, DevCamera cam,
    double t, double scale, float* __restrict__ g4, float* __restrict__ g3, float* __restrict__ sn4,
    float* __restrict__ sn3, float* __restrict__ gn4, float* __restrict__ gn3, float* __restrict__ cnt4,
    float* __restrict__ cnt3, const double* __restrict__ conic_src, int conic_stride,
    const float4* __restrict__ ddir, int first) {
    pdl_wait();  // launched with launch_pdl
    // one thread per Gaussian in pool order (coalesced SoA parameter and
    // gradient rows); the splat's accumulators are found through the
    // gid -> depth-sorted index map written by the gather kernel
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= N) return;
    const uint32_t j = sorted_of_gid[gid];
    if (j == 0xffffffffu) return;  // not visible in this view
    const float* acc = accum + (size_t)j * acc_stride;
    const double d_rgb[3] = {acc[0], acc[1], acc[2]};
    const double d_alpha = acc[3];
    if (d_rgb[0] == 0.0 && d_rgb[1] == 0.0 && d_rgb[2] == 0.0 && d_alpha == 0.0 && acc[4] == 0.0f &&
        acc[5] == 0.0f && acc[6] == 0.0f && acc[7] == 0.0f && acc[8] == 0.0f)
        return;  // untouched (backward.cpp:226)
    const bool dyn = gid < n4;
    const int i = dyn ? gid : gid - n4;
    const float* P = dyn ? p4 : p3;
    const int64_t cap = dyn ? cap4 : cap3;
    // all geometry rows loaded up front (independent loads in flight together)
    float pg[R4_SH];
#pragma unroll
    for (int r = 0; r < R4_SH; ++r) pg[r] = (dyn || r < R3_SH) ? P[(int64_t)r * cap + i] : 0.0f;
    auto prm = [&](int row) { return (double)pg[row]; };
    const double* cn = conic_src + (size_t)j * conic_stride;
    const double C[2][2] = {{cn[0], cn[1]}, {cn[2], cn[3]}};
    // K6's conic-free sums -> d_screen = alpha * C . (sum h dx, sum h dy) and
    // d_conic = -alpha/2 * sum h d d^T (backward.cpp:212-221)
    const double ag = cn[4];  // SplatRec::alpha follows c11
    const double d_screen[2] = {ag * (C[0][0] * acc[4] + C[0][1] * acc[5]), ag * (C[1][0] * acc[4] + C[1][1] * acc[5])};
    const double hc = -0.5 * ag;
    const double dC[2][2] = {{hc * acc[6], hc * acc[7]}, {hc * acc[7], hc * acc[8]}};

    // ---- forward intermediates
    double mean3[3], cov3[3][3], weight = 1.0, opl, R4[4][4], es[4], ql[4], qr[4], q3[4], cross[3], s44 = 1.0, dt = 0.0;
    bool clamped;
    if (dyn) {
        for (int k = 0; k < 4; ++k) {
            ql[k] = prm(R4_QL + k);
            qr[k] = prm(R4_QR + k);
            es[k] = exp(prm(R4_LS + k));
        }
        double L[4][4], R[4][4];
        isoL(ql, L);
        isoR(qr, R);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += L[a][k] * R[k][b];
                R4[a][b] = s;
            }
        double M[4][4], S4[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) M[a][b] = R4[a][b] * es[b];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += M[a][k] * M[b][k];
                S4[a][b] = s;
            }
        s44 = S4[3][3];
        for (int k = 0; k < 3; ++k) cross[k] = S4[k][3];
        dt = t - prm(R4_MT);
        for (int k = 0; k < 3; ++k) mean3[k] = prm(R4_MEAN + k) + cross[k] * (dt / s44);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) cov3[a][b] = S4[a][b] - cross[a] * cross[b] / s44;
        weight = exp(-0.5 * dt * dt / s44);
        opl = prm(R4_OP);
        clamped = sigmoid(opl) * weight >= kAlphaClamp;
    } else {
        for (int k = 0; k < 4; ++k) q3[k] = prm(R3_Q + k);
        for (int k = 0; k < 3; ++k) {
            es[k] = exp(prm(R3_LS + k));
            mean3[k] = prm(R3_MEAN + k);
        }
        const double w = q3[0], x = q3[1], y = q3[2], z = q3[3];
        const double Rm[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)},
                                 {2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)},
                                 {2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)}};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k) s += Rm[a][k] * es[k] * Rm[b][k] * es[k];
                cov3[a][b] = s;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) R4[a][b] = Rm[a][b];  // reuse storage for the 3x3 rotation
        opl = prm(R3_OP);
        clamped = sigmoid(opl) >= kAlphaClamp;
    }
    double cp[3];
    for (int a = 0; a < 3; ++a) cp[a] = cam.R[a * 3] * mean3[0] + cam.R[a * 3 + 1] * mean3[1] + cam.R[a * 3 + 2] * mean3[2] + cam.t[a];
    const double z = cp[2], xq = cp[0], yq = cp[1];
    const double J[2][3] = {{cam.fx / z, 0.0, -cam.fx * xq / (z * z)}, {0.0, cam.fy / z, -cam.fy * yq / (z * z)}};
    double Tm[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) Tm[a][k] = J[a][0] * cam.R[k] + J[a][1] * cam.R[3 + k] + J[a][2] * cam.R[6 + k];

    // ---- conic -> cov2 -> cov3 / camera mean (backward.cpp:231-250)
    double CdC[2][2], d_cov2[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) CdC[a][b] = C[a][0] * dC[0][b] + C[a][1] * dC[1][b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) d_cov2[a][b] = -(CdC[a][0] * C[0][b] + CdC[a][1] * C[1][b]);
    double dT[2][3];  // d_cov2 * T
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) dT[a][k] = d_cov2[a][0] * Tm[0][k] + d_cov2[a][1] * Tm[1][k];
    double d_cov3[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_cov3[a][b] = Tm[0][a] * dT[0][b] + Tm[1][a] * dT[1][b];
    double d_tmat[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) d_tmat[a][k] = 2.0 * (dT[a][0] * cov3[0][k] + dT[a][1] * cov3[1][k] + dT[a][2] * cov3[2][k]);
    double d_jac[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k)
            d_jac[a][k] = d_tmat[a][0] * cam.R[k * 3] + d_tmat[a][1] * cam.R[k * 3 + 1] + d_tmat[a][2] * cam.R[k * 3 + 2];
    double d_cp[3];
    for (int k = 0; k < 3; ++k) d_cp[k] = J[0][k] * d_screen[0] + J[1][k] * d_screen[1];
    const double fx = cam.fx, fy = cam.fy;
    d_cp[0] += d_jac[0][2] * (-fx / (z * z));
    d_cp[1] += d_jac[1][2] * (-fy / (z * z));
    d_cp[2] += d_jac[0][0] * (-fx / (z * z)) + d_jac[1][1] * (-fy / (z * z)) + d_jac[0][2] * (2.0 * fx * xq / (z * z * z)) +
               d_jac[1][2] * (2.0 * fy * yq / (z * z * z));
    double d_mean3[3];
    for (int k = 0; k < 3; ++k) d_mean3[k] = cam.R[k] * d_cp[0] + cam.R[3 + k] * d_cp[1] + cam.R[6 + k] * d_cp[2];

    // ---- colour path (backward.cpp:252-273)
    double v[3] = {mean3[0] - cam.pos[0], mean3[1] - cam.pos[1], mean3[2] - cam.pos[2]};
    const double vd = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    double dir[3] = {0.0, 0.0, 1.0};
    if (vd > 0.0)
        for (int k = 0; k < 3; ++k) dir[k] = v[k] / vd;
    float* G = dyn ? g4 : g3;
    // Gradient rows are read-modify-written in one batch at the end (all
    // loads before the stores): the row pointers alias as far as the compiler
    // knows, so one-at-a-time RMW would serialise the memory latencies.
    float gacc[R4_SH];
#pragma unroll
    for (int r = 0; r < R4_SH; ++r) gacc[r] = 0.0f;
    auto gadd = [&](int row, double val) { gacc[row] = (float)(scale * val); };
    // d(loss)/d(view direction) from the SH backward (K7b, sh_bwd_kernel)
    const float4 dd = ddir[gid];
    const double d_dir[3] = {dd.x, dd.y, dd.z};
    if (vd > 0.0)
        for (int a = 0; a < 3; ++a) {
            double s = 0.0;
            for (int b = 0; b < 3; ++b) s += ((a == b ? 1.0 : 0.0) - dir[a] * dir[b]) / vd * d_dir[b];
            d_mean3[a] += s;
        }
    const double screen_norm = sqrt(d_screen[0] * d_screen[0] + d_screen[1] * d_screen[1]);
    double dS[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dS[a][b] = 0.5 * (d_cov3[a][b] + d_cov3[b][a]);
    const double sg = sigmoid(opl);

    if (!dyn) {
        for (int k = 0; k < 3; ++k) gadd(R3_MEAN + k, d_mean3[k]);
        if (!clamped) gadd(R3_OP, d_alpha * sg * (1.0 - sg));
        double m[3][3], dm[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) m[a][b] = R4[a][b] * es[b];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dm[a][b] = 2.0 * (dS[a][0] * m[0][b] + dS[a][1] * m[1][b] + dS[a][2] * m[2][b]);
        for (int k = 0; k < 3; ++k) gadd(R3_LS + k, dm[0][k] * m[0][k] + dm[1][k] * m[1][k] + dm[2][k] * m[2][k]);
        double dR[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dR[a][b] = dm[a][b] * es[b];
        const double w = q3[0], x = q3[1], y = q3[2], zz = q3[3];
        // drot3_dq (backward.cpp:54-72), contracted with dR
        const double D[4][3][3] = {{{0, -zz, y}, {zz, 0, -x}, {-y, x, 0}},
                                   {{0, y, zz}, {y, -2 * x, -w}, {zz, w, -2 * x}},
                                   {{-2 * y, x, w}, {x, 0, zz}, {-w, zz, -2 * y}},
                                   {{-2 * zz, -w, x}, {w, -2 * zz, y}, {x, y, 0}}};
        double dq[4];
        for (int k = 0; k < 4; ++k) {
            double s = 0.0;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) s += dR[a][b] * 2.0 * D[k][a][b];
            dq[k] = s;
        }
        const double qd = q3[0] * dq[0] + q3[1] * dq[1] + q3[2] * dq[2] + q3[3] * dq[3];
        for (int k = 0; k < 4; ++k) gadd(R3_Q + k, dq[k] - qd * q3[k]);
        sn3[i] = (float)screen_norm;
        if (screen_norm > 0.0) {
            gn3[i] += (float)screen_norm;
            cnt3[i] += 1.0f;
        }
        float old[R3_SH];
#pragma unroll
        for (int r = 0; r < R3_SH; ++r) old[r] = first ? 0.0f : G[(int64_t)r * cap + i];
#pragma unroll
        for (int r = 0; r < R3_SH; ++r) G[(int64_t)r * cap + i] = old[r] + gacc[r];
    } else {
        double d_weight = 0.0;
        if (!clamped) {
            gadd(R4_OP, d_alpha * weight * sg * (1.0 - sg));
            d_weight += d_alpha * sg;
        }
        for (int k = 0; k < 3; ++k) gadd(R4_MEAN + k, d_mean3[k]);
        const double dmc = d_mean3[0] * cross[0] + d_mean3[1] * cross[1] + d_mean3[2] * cross[2];
        gadd(R4_MT, -dmc / s44 + d_weight * weight * dt / s44);
        double sc[3];
        for (int a = 0; a < 3; ++a) sc[a] = dS[a][0] * cross[0] + dS[a][1] * cross[1] + dS[a][2] * cross[2];
        double d_cross[3];
        for (int a = 0; a < 3; ++a) d_cross[a] = d_mean3[a] * (dt / s44) - 2.0 * sc[a] / s44;
        const double csc = cross[0] * sc[0] + cross[1] * sc[1] + cross[2] * sc[2];
        const double d_s44 = -dmc * dt / (s44 * s44) + csc / (s44 * s44) + d_weight * weight * 0.5 * dt * dt / (s44 * s44);
        double d4[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) d4[a][b] = 0.0;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) d4[a][b] = dS[a][b];
        for (int a = 0; a < 3; ++a) d4[a][3] = d_cross[a];
        d4[3][3] = d_s44;
        double m4[4][4], dm4[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) m4[a][b] = R4[a][b] * es[b];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += (d4[a][k] + d4[k][a]) * m4[k][b];
                dm4[a][b] = s;
            }
        for (int k = 0; k < 4; ++k)
            gadd(R4_LS + k, dm4[0][k] * m4[0][k] + dm4[1][k] * m4[1][k] + dm4[2][k] * m4[2][k] + dm4[3][k] * m4[3][k]);
        double dR4[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) dR4[a][b] = dm4[a][b] * es[b];
        double L[4][4], R[4][4];
        isoL(ql, L);
        isoR(qr, R);
        double dL[4][4], dR[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double x = 0.0, y = 0.0;
                for (int k = 0; k < 4; ++k) {
                    x += dR4[a][k] * R[b][k];
                    y += L[k][a] * dR4[k][b];
                }
                dL[a][b] = x;
                dR[a][b] = y;
            }
        double dql[4], dqr[4];
        for (int k = 0; k < 4; ++k) {
            double ek[4] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0, k == 3 ? 1.0 : 0.0};
            double le[4][4], re[4][4];
            isoL(ek, le);
            isoR(ek, re);
            double x = 0.0, y = 0.0;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) {
                    x += dL[a][b] * le[a][b];
                    y += dR[a][b] * re[a][b];
                }
            dql[k] = x;
            dqr[k] = y;
        }
        const double dl = ql[0] * dql[0] + ql[1] * dql[1] + ql[2] * dql[2] + ql[3] * dql[3];
        const double dr = qr[0] * dqr[0] + qr[1] * dqr[1] + qr[2] * dqr[2] + qr[3] * dqr[3];
        for (int k = 0; k < 4; ++k) {
            gadd(R4_QL + k, dql[k] - dl * ql[k]);
            gadd(R4_QR + k, dqr[k] - dr * qr[k]);
        }
        sn4[i] = (float)screen_norm;
        if (screen_norm > 0.0) {
            gn4[i] += (float)screen_norm;
            cnt4[i] += 1.0f;
        }
        float old[R4_SH];
#pragma unroll
        for (int r = 0; r < R4_SH; ++r) old[r] = first ? 0.0f : G[(int64_t)r * cap + i];
#pragma unroll
        for (int r = 0; r < R4_SH; ++r) G[(int64_t)r * cap + i] = old[r] + gacc[r];
    }
}

// K7b: SH colour backward (backward.cpp:252-273), one thread per visible
// Gaussian, FP32: dL/dSH_k = scale * Y_k(dir) * dL/drgb (zero on clamped
// channels) into the SH gradient rows, and dL/d(dir) = sum_k (dL/drgb . SH_k)
// dY_k/d(dir) for K7 (which chains it into the mean).  The view direction and
// the clamped-channel mask were recorded by K1.  Split from K7 so the
// FP64 geometry kernel carries no SH state (occupancy) and the 48-row
// coefficient / gradient traffic runs at high memory-level parallelism.
__global__ void __launch_bounds__(128) sh_bwd_kernel(int N, const uint32_t* __restrict__ sorted_of_gid,
                                                     const float* __restrict__ accum, int acc_stride, int n4,
                                                     const float* __restrict__ p4, int64_t cap4,
                                                     const float* __restrict__ p3, int64_t cap3, int deg, float scale,
                                                     float* __restrict__ g4, float* __restrict__ g3,
                                                     const ShRec* __restrict__ shrec, float4* __restrict__ ddir,
                                                     int first) {
    pdl_wait();  // launched with launch_pdl
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= N) return;
    const uint32_t j = sorted_of_gid[gid];
    if (j == 0xffffffffu) return;  // not visible in this view
    const float* acc = accum + (size_t)j * acc_stride;
    const float4 a03 = *reinterpret_cast<const float4*>(acc);
    const float4 a47 = *reinterpret_cast<const float4*>(acc + 4);
    if (a03.x == 0.f && a03.y == 0.f && a03.z == 0.f && a03.w == 0.f && a47.x == 0.f && a47.y == 0.f &&
        a47.z == 0.f && a47.w == 0.f && acc[8] == 0.f)
        return;  // untouched (backward.cpp:226): K7 skips it too
    const bool dyn = gid < n4;
    const int i = dyn ? gid : gid - n4;
    float* Gs = (dyn ? g4 : g3) + i;
    const int64_t cap = dyn ? cap4 : cap3;
    const int shrow = dyn ? R4_SH : R3_SH;
    const ShRec sr = shrec[gid];
    const float df[3] = {sr.dir.x, sr.dir.y, sr.dir.z};
    const uint32_t clamped = __float_as_uint(sr.dir.w);
    const float d_rgb[3] = {a03.x, a03.y, a03.z};
    float drr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) drr[c] = ((clamped >> c) & 1u) ? 0.0f : d_rgb[c];
    // dL/d(direction) = sum_c drr_c * d rgb_c / d direction (K1's Jacobian)
    ddir[gid] = make_float4(fmaf(drr[0], sr.j[0].x, fmaf(drr[1], sr.j[1].x, drr[2] * sr.j[2].x)),
                            fmaf(drr[0], sr.j[0].y, fmaf(drr[1], sr.j[1].y, drr[2] * sr.j[2].y)),
                            fmaf(drr[0], sr.j[0].z, fmaf(drr[1], sr.j[1].z, drr[2] * sr.j[2].z)), 0.f);
    float basis[16];
    sh_basis_f(df, deg, basis);
    const int K = sh_count(deg);
    float* G = Gs + (int64_t)shrow * cap;
    if (first) {  // the gradient buffer is known to be zero: plain stores
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < K)
#pragma unroll
                for (int c = 0; c < 3; ++c) G[(int64_t)(3 * k + c) * cap] = scale * (basis[k] * drr[c]);
        return;
    }
#pragma unroll
    for (int k0 = 0; k0 < 16; k0 += 4) {
        // 4 coefficients (12 rows): loads first, then the stores
        float gv[12];
#pragma unroll
        for (int u = 0; u < 12; ++u)
            if (k0 + u / 3 < K) gv[u] = G[(int64_t)(3 * k0 + u) * cap];
#pragma unroll
        for (int u = 0; u < 12; ++u)
            if (k0 + u / 3 < K) G[(int64_t)(3 * k0 + u) * cap] = fmaf(scale, basis[k0 + u / 3] * drr[u % 3], gv[u]);
    }
}

}  // namespace hgs
