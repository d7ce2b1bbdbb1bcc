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

// Forward intermediates of one Gaussian (FP64), shared by the value and the
// error-bound evaluation of the chain.
struct Geo {
    bool dyn, clamped;
    double C[2][2], ag;                   // conic, alpha
    double cov3[3][3], J[2][3], Tm[2][3];  // slice covariance, projection Jacobian, J W
    double z, xq, yq;                      // camera-space mean
    double dir[3], vd;                     // view direction, distance
    double R4[4][4], es[4];                // 4D rotation (3D: rotation in [0..2][0..2]), exp(scales)
    double q[4], ql[4], qr[4];
    double cross[3], s44, dt, weight, sg;
    double i44, iz, ivd;  // 1/s44, 1/z, 1/|v| (K7 is toleranced: one reciprocal per divisor)
};

__device__ __forceinline__ void geometry(Geo& g, const float pg[R4_SH], const double* cn, const DevCamera& cam,
                                         double t, bool dyn) {
    auto prm = [&](int row) { return (double)pg[row]; };
    g.dyn = dyn;
    g.C[0][0] = cn[0];
    g.C[0][1] = cn[1];
    g.C[1][0] = cn[2];
    g.C[1][1] = cn[3];
    g.ag = cn[4];  // SplatRec::alpha follows c11
    double mean3[3], opl;
    g.weight = 1.0;
    g.s44 = 1.0;
    g.i44 = 1.0;
    g.dt = 0.0;
    if (dyn) {
        for (int k = 0; k < 4; ++k) {
            g.ql[k] = prm(R4_QL + k);
            g.qr[k] = prm(R4_QR + k);
            g.es[k] = exp(prm(R4_LS + k));
        }
        double L[4][4], R[4][4];
        isoL(g.ql, L);
        isoR(g.qr, R);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += L[a][k] * R[k][b];
                g.R4[a][b] = s;
            }
        double M[4][4], S4[4][4];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) M[a][b] = g.R4[a][b] * g.es[b];
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
                double s = 0.0;
                for (int k = 0; k < 4; ++k) s += M[a][k] * M[b][k];
                S4[a][b] = s;
            }
        g.s44 = S4[3][3];
        for (int k = 0; k < 3; ++k) g.cross[k] = S4[k][3];
        g.dt = t - prm(R4_MT);
        g.i44 = 1.0 / g.s44;
        const double f = g.dt * g.i44;
        for (int k = 0; k < 3; ++k) mean3[k] = prm(R4_MEAN + k) + g.cross[k] * f;
        for (int a = 0; a < 3; ++a)
            for (int b = a; b < 3; ++b) {
                g.cov3[a][b] = S4[a][b] - g.cross[a] * g.cross[b] * g.i44;
                g.cov3[b][a] = g.cov3[a][b];
            }
        g.weight = exp(-0.5 * g.dt * g.dt * g.i44);
        opl = prm(R4_OP);
        g.clamped = sigmoid(opl) * g.weight >= kAlphaClamp;
    } else {
        for (int k = 0; k < 4; ++k) g.q[k] = prm(R3_Q + k);
        for (int k = 0; k < 3; ++k) {
            g.es[k] = exp(prm(R3_LS + k));
            mean3[k] = prm(R3_MEAN + k);
        }
        const double w = g.q[0], x = g.q[1], y = g.q[2], z = g.q[3];
        const double Rm[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)},
                                 {2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)},
                                 {2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)}};
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k) s += Rm[a][k] * g.es[k] * Rm[b][k] * g.es[k];
                g.cov3[a][b] = s;
            }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) g.R4[a][b] = Rm[a][b];  // reuse storage for the 3x3 rotation
        opl = prm(R3_OP);
        g.clamped = sigmoid(opl) >= kAlphaClamp;
    }
    g.sg = sigmoid(opl);
    double cp[3];
    for (int a = 0; a < 3; ++a)
        cp[a] = cam.R[a * 3] * mean3[0] + cam.R[a * 3 + 1] * mean3[1] + cam.R[a * 3 + 2] * mean3[2] + cam.t[a];
    g.z = cp[2];
    g.xq = cp[0];
    g.yq = cp[1];
    g.iz = 1.0 / g.z;
    const double iz = g.iz, iz2 = iz * iz;
    g.J[0][0] = cam.fx * iz;
    g.J[0][1] = 0.0;
    g.J[0][2] = -cam.fx * g.xq * iz2;
    g.J[1][0] = 0.0;
    g.J[1][1] = cam.fy * iz;
    g.J[1][2] = -cam.fy * g.yq * iz2;
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k)
            g.Tm[a][k] = g.J[a][0] * cam.R[k] + g.J[a][1] * cam.R[3 + k] + g.J[a][2] * cam.R[6 + k];
    const double v[3] = {mean3[0] - cam.pos[0], mean3[1] - cam.pos[1], mean3[2] - cam.pos[2]};
    g.vd = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    g.dir[0] = 0.0;
    g.dir[1] = 0.0;
    g.dir[2] = 1.0;
    g.ivd = 0.0;
    if (g.vd > 0.0) {
        g.ivd = 1.0 / g.vd;
        for (int k = 0; k < 3; ++k) g.dir[k] = v[k] * g.ivd;
    }
}

// The accumulator-dependent part of backward.cpp:224-354: K6's conic-free
// sums acc[3..8] and d loss / d view direction -> the geometry rows of the
// Gaussian's gradient (out[row], rows not written stay 0) and d_screen.
template <typename T>
__device__ __forceinline__ void chain(const Geo& g, const DevCamera& cam, const T acc[9], const T d_dir[3],
                                      T out[R4_SH], T d_screen[2]) {
    for (int r = 0; r < R4_SH; ++r) out[r] = T(0.0);
    const double(&C)[2][2] = g.C;
    // K6's conic-free sums -> d_screen = alpha * C . (sum h dx, sum h dy) and
    // d_conic = -alpha/2 * sum h d d^T (backward.cpp:212-221)
    d_screen[0] = g.ag * (C[0][0] * acc[4] + C[0][1] * acc[5]);
    d_screen[1] = g.ag * (C[1][0] * acc[4] + C[1][1] * acc[5]);
    const double hc = -0.5 * g.ag;
    const T dC[2][2] = {{hc * acc[6], hc * acc[7]}, {hc * acc[7], hc * acc[8]}};
    const T d_alpha = acc[3];

    // ---- conic -> cov2 -> cov3 / camera mean (backward.cpp:231-250)
    T CdC[2][2], d_cov2[2][2];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) CdC[a][b] = C[a][0] * dC[0][b] + C[a][1] * dC[1][b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) d_cov2[a][b] = -(CdC[a][0] * C[0][b] + CdC[a][1] * C[1][b]);
    T dT[2][3];  // d_cov2 * T
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) dT[a][k] = d_cov2[a][0] * g.Tm[0][k] + d_cov2[a][1] * g.Tm[1][k];
    T d_cov3[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d_cov3[a][b] = g.Tm[0][a] * dT[0][b] + g.Tm[1][a] * dT[1][b];
    T d_tmat[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k)
            d_tmat[a][k] = 2.0 * (dT[a][0] * g.cov3[0][k] + dT[a][1] * g.cov3[1][k] + dT[a][2] * g.cov3[2][k]);
    T d_jac[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k)
            d_jac[a][k] = d_tmat[a][0] * cam.R[k * 3] + d_tmat[a][1] * cam.R[k * 3 + 1] + d_tmat[a][2] * cam.R[k * 3 + 2];
    T d_cp[3];
    for (int k = 0; k < 3; ++k) d_cp[k] = g.J[0][k] * d_screen[0] + g.J[1][k] * d_screen[1];
    const double fx = cam.fx, fy = cam.fy, iz = g.iz, xq = g.xq, yq = g.yq;
    const double iz2 = iz * iz, iz3 = iz2 * iz;
    d_cp[0] += d_jac[0][2] * (-fx * iz2);
    d_cp[1] += d_jac[1][2] * (-fy * iz2);
    d_cp[2] += d_jac[0][0] * (-fx * iz2) + d_jac[1][1] * (-fy * iz2) + d_jac[0][2] * (2.0 * fx * xq * iz3) +
               d_jac[1][2] * (2.0 * fy * yq * iz3);
    T d_mean3[3];
    for (int k = 0; k < 3; ++k) d_mean3[k] = cam.R[k] * d_cp[0] + cam.R[3 + k] * d_cp[1] + cam.R[6 + k] * d_cp[2];
    // ---- colour path (backward.cpp:252-273): d loss / d view direction
    if (g.vd > 0.0)
        for (int a = 0; a < 3; ++a) {
            T s = T(0.0);
            for (int b = 0; b < 3; ++b) s += ((a == b ? 1.0 : 0.0) - g.dir[a] * g.dir[b]) * g.ivd * d_dir[b];
            d_mean3[a] += s;
        }
    T dS[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dS[a][b] = 0.5 * (d_cov3[a][b] + d_cov3[b][a]);
    const double sg = g.sg;

    if (!g.dyn) {
        for (int k = 0; k < 3; ++k) out[R3_MEAN + k] = d_mean3[k];
        if (!g.clamped) out[R3_OP] = d_alpha * sg * (1.0 - sg);
        double m[3][3];
        T dm[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) m[a][b] = g.R4[a][b] * g.es[b];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dm[a][b] = 2.0 * (dS[a][0] * m[0][b] + dS[a][1] * m[1][b] + dS[a][2] * m[2][b]);
        for (int k = 0; k < 3; ++k) out[R3_LS + k] = dm[0][k] * m[0][k] + dm[1][k] * m[1][k] + dm[2][k] * m[2][k];
        T dR[3][3];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) dR[a][b] = dm[a][b] * g.es[b];
        const double w = g.q[0], x = g.q[1], y = g.q[2], zz = g.q[3];
        // drot3_dq (backward.cpp:54-72) contracted with dR, its zero entries dropped
        //   D0 = {{0, -z, y}, {z, 0, -x}, {-y, x, 0}}      D1 = {{0, y, z}, {y, -2x, -w}, {z, w, -2x}}
        //   D2 = {{-2y, x, w}, {x, 0, z}, {-w, z, -2y}}     D3 = {{-2z, -w, x}, {w, -2z, y}, {x, y, 0}}
        const T dq[4] = {
            2.0 * (-zz * dR[0][1] + y * dR[0][2] + zz * dR[1][0] - x * dR[1][2] - y * dR[2][0] + x * dR[2][1]),
            2.0 * (y * dR[0][1] + zz * dR[0][2] + y * dR[1][0] - 2 * x * dR[1][1] - w * dR[1][2] + zz * dR[2][0] +
                   w * dR[2][1] - 2 * x * dR[2][2]),
            2.0 * (-2 * y * dR[0][0] + x * dR[0][1] + w * dR[0][2] + x * dR[1][0] + zz * dR[1][2] - w * dR[2][0] +
                   zz * dR[2][1] - 2 * y * dR[2][2]),
            2.0 * (-2 * zz * dR[0][0] - w * dR[0][1] + x * dR[0][2] + w * dR[1][0] - 2 * zz * dR[1][1] +
                   y * dR[1][2] + x * dR[2][0] + y * dR[2][1])};
        const T qd = g.q[0] * dq[0] + g.q[1] * dq[1] + g.q[2] * dq[2] + g.q[3] * dq[3];
        for (int k = 0; k < 4; ++k) out[R3_Q + k] = dq[k] - qd * g.q[k];
        return;
    }
    T d_weight = T(0.0);
    if (!g.clamped) {
        out[R4_OP] = d_alpha * g.weight * sg * (1.0 - sg);
        d_weight += d_alpha * sg;
    }
    for (int k = 0; k < 3; ++k) out[R4_MEAN + k] = d_mean3[k];
    const double i44 = g.i44, dt = g.dt, weight = g.weight, i44s = i44 * i44;
    const double(&cross)[3] = g.cross;
    const T dmc = d_mean3[0] * cross[0] + d_mean3[1] * cross[1] + d_mean3[2] * cross[2];
    out[R4_MT] = -dmc * i44 + d_weight * weight * dt * i44;
    T sc[3];
    for (int a = 0; a < 3; ++a) sc[a] = dS[a][0] * cross[0] + dS[a][1] * cross[1] + dS[a][2] * cross[2];
    T d_cross[3];
    for (int a = 0; a < 3; ++a) d_cross[a] = d_mean3[a] * (dt * i44) - 2.0 * sc[a] * i44;
    const T csc = cross[0] * sc[0] + cross[1] * sc[1] + cross[2] * sc[2];
    const T d_s44 = -dmc * dt * i44s + csc * i44s + d_weight * weight * 0.5 * dt * dt * i44s;
    T d4[4][4];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) d4[a][b] = T(0.0);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) d4[a][b] = dS[a][b];
    for (int a = 0; a < 3; ++a) d4[a][3] = d_cross[a];
    d4[3][3] = d_s44;
    double m4[4][4];
    T dm4[4][4];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) m4[a][b] = g.R4[a][b] * g.es[b];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            T s = T(0.0);
            for (int k = 0; k < 4; ++k) s += (d4[a][k] + d4[k][a]) * m4[k][b];
            dm4[a][b] = s;
        }
    for (int k = 0; k < 4; ++k)
        out[R4_LS + k] = dm4[0][k] * m4[0][k] + dm4[1][k] * m4[1][k] + dm4[2][k] * m4[2][k] + dm4[3][k] * m4[3][k];
    T dR4[4][4];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) dR4[a][b] = dm4[a][b] * g.es[b];
    double L[4][4], R[4][4];
    isoL(g.ql, L);
    isoR(g.qr, R);
    T dL[4][4], dR[4][4];
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            T x = T(0.0), y = T(0.0);
            for (int k = 0; k < 4; ++k) {
                x += dR4[a][k] * R[b][k];
                y += L[k][a] * dR4[k][b];
            }
            dL[a][b] = x;
            dR[a][b] = y;
        }
    // d/dq_k of the isoclinic factors contracted with dL, dR: isoL(e_k) and
    // isoR(e_k) are signed permutation matrices (isoL / isoR above), so each
    // contraction is 4 signed terms (the zero products of the dense form are
    // not folded by the compiler: 0 * x is not 0 for a NaN x)
    const T dql[4] = {dL[0][0] + dL[1][1] + dL[2][2] + dL[3][3], -dL[0][1] + dL[1][0] - dL[2][3] + dL[3][2],
                      -dL[0][2] + dL[1][3] + dL[2][0] - dL[3][1], -dL[0][3] - dL[1][2] + dL[2][1] + dL[3][0]};
    const T dqr[4] = {dR[0][0] + dR[1][1] + dR[2][2] + dR[3][3], -dR[0][1] + dR[1][0] + dR[2][3] - dR[3][2],
                      -dR[0][2] - dR[1][3] + dR[2][0] + dR[3][1], -dR[0][3] + dR[1][2] - dR[2][1] + dR[3][0]};
    const double(&ql)[4] = g.ql;
    const double(&qr)[4] = g.qr;
    const T dl = ql[0] * dql[0] + ql[1] * dql[1] + ql[2] * dql[2] + ql[3] * dql[3];
    const T dr = qr[0] * dqr[0] + qr[1] * dqr[1] + qr[2] * dqr[2] + qr[3] * dqr[3];
    for (int k = 0; k < 4; ++k) {
        out[R4_QL + k] = dql[k] - dl * ql[k];
        out[R4_QR + k] = dqr[k] - dr * qr[k];
    }
}

// FP64 colour of a Gaussian seen from the camera (sh.cpp:73-83 with the
// view direction of raster.cpp:83-85): raw channel values (before the
// [0,1] clamp) and the SH basis.  Exact backward mode only.
__device__ inline void sh_colour64(const float* P, int64_t cap, int i, int shrow, int deg, const double dir[3],
                                   double raw[3], double basis[16]) {
    sh_basis_t<double>(dir, deg, basis);
    const int K = sh_count(deg);
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int k = 0; k < K; ++k) acc += (double)P[(int64_t)(shrow + 3 * k + c) * cap + i] * basis[k];
        raw[c] = acc + 0.5;
    }
}

}  // namespace

// K7 body.  kExact (exact backward mode, hgs_set_exact_backward): the
// accumulators come from the all-pixel FP64 walk, and the SH rows and
// d loss / d view direction are formed here in FP64 from the SH
// coefficients (K7b does not run).
template <bool kExact>
__device__ __forceinline__ void gaussian_bwd_body(
    int N, const uint32_t* __restrict__ sorted_of_gid, const acc_t* __restrict__ accum, int acc_stride, int n4,
    const float* __restrict__ p4, int64_t cap4, const float* __restrict__ p3, int64_t cap3, int deg, DevCamera cam,
    double t, double scale, float* __restrict__ g4, float* __restrict__ g3, float* __restrict__ sn4,
    float* __restrict__ sn3, float* __restrict__ gn4, float* __restrict__ gn3, float* __restrict__ cnt4,
    float* __restrict__ cnt3, const double* __restrict__ conic_src, int conic_stride,
    const float4* __restrict__ ddir, int first) {
    // one thread per Gaussian in pool order (coalesced SoA parameter and
    // gradient rows); the splat's accumulators are found through the
    // gid -> depth-sorted index map written by the gather kernel
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= N) return;
    const uint32_t j = sorted_of_gid[gid];
    if (j == 0xffffffffu) return;  // not visible in this view
    HGS_DCHECK(j < g_chk.splats);
    const acc_t* acc = accum + (size_t)j * acc_stride;
    double av[9];
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const double2 p = *reinterpret_cast<const double2*>(acc + k);
        av[k] = p.x;
        av[k + 1] = p.y;
    }
    av[8] = acc[8];
    if (av[0] == 0.0 && av[1] == 0.0 && av[2] == 0.0 && av[3] == 0.0 && av[4] == 0.0 && av[5] == 0.0 &&
        av[6] == 0.0 && av[7] == 0.0 && av[8] == 0.0)
        return;  // untouched (backward.cpp:226)
    const bool dyn = gid < n4;
    const int i = dyn ? gid : gid - n4;
    const float* P = dyn ? p4 : p3;
    const int64_t cap = dyn ? cap4 : cap3;
    // all geometry rows loaded up front (independent loads in flight together)
    float pg[R4_SH];
#pragma unroll
    for (int r = 0; r < R4_SH; ++r) pg[r] = (dyn || r < R3_SH) ? P[(int64_t)r * cap + i] : 0.0f;
    const double* cn = conic_src + (size_t)j * conic_stride;
    Geo g;
    geometry(g, pg, cn, cam, t, dyn);
    float* G = dyn ? g4 : g3;
    double d_dir[3];
    if (!kExact) {
        // d(loss)/d(view direction) from the SH backward (K7b, sh_bwd_kernel)
        const float4 dd = ddir[gid];
        d_dir[0] = dd.x;
        d_dir[1] = dd.y;
        d_dir[2] = dd.z;
    } else {
        // the SH backward of backward.cpp:252-273 in FP64
        const int shrow = dyn ? R4_SH : R3_SH;
        double raw[3], basis[16];
        sh_colour64(P, cap, i, shrow, deg, g.dir, raw, basis);
        double drr[3];
        for (int c = 0; c < 3; ++c) drr[c] = (raw[c] < 0.0 || raw[c] > 1.0) ? 0.0 : av[c];
        const int K = sh_count(deg);
        d_dir[0] = d_dir[1] = d_dir[2] = 0.0;
        for (int c = 0; c < 3; ++c) {
            double w[16];
            for (int k = 0; k < 16; ++k) w[k] = k < K ? (double)P[(int64_t)(shrow + 3 * k + c) * cap + i] : 0.0;
            double gd[3];
            sh_dir_grad_t<double>(g.dir, deg, w, gd);
            for (int b = 0; b < 3; ++b) d_dir[b] += drr[c] * gd[b];
        }
        float* Gs = G + (int64_t)shrow * cap + i;
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) {
                const double v = scale * (basis[k] * drr[c]);
                float* dst = Gs + (int64_t)(3 * k + c) * cap;
                *dst = first ? (float)v : *dst + (float)v;
            }
    }
    double out[R4_SH], d_screen[2];
    chain<double>(g, cam, av, d_dir, out, d_screen);
    const double screen_norm = sqrt(d_screen[0] * d_screen[0] + d_screen[1] * d_screen[1]);
    // Gradient rows are read-modify-written in one batch at the end (all
    // loads before the stores): the row pointers alias as far as the compiler
    // knows, so one-at-a-time RMW would serialise the memory latencies.
    float gacc[R4_SH];
#pragma unroll
    for (int r = 0; r < R4_SH; ++r) gacc[r] = (float)(scale * out[r]);
    float* sn = dyn ? sn4 : sn3;
    float* gn = dyn ? gn4 : gn3;
    float* cntp = dyn ? cnt4 : cnt3;
    sn[i] = (float)screen_norm;
    if (screen_norm > 0.0) {
        gn[i] += (float)screen_norm;
        cntp[i] += 1.0f;
    }
    if (dyn) {
        float old[R4_SH];
#pragma unroll
        for (int r = 0; r < R4_SH; ++r) old[r] = first ? 0.0f : G[(int64_t)r * cap + i];
#pragma unroll
        for (int r = 0; r < R4_SH; ++r) G[(int64_t)r * cap + i] = old[r] + gacc[r];
    } else {
        float old[R3_SH];
#pragma unroll
        for (int r = 0; r < R3_SH; ++r) old[r] = first ? 0.0f : G[(int64_t)r * cap + i];
#pragma unroll
        for (int r = 0; r < R3_SH; ++r) G[(int64_t)r * cap + i] = old[r] + gacc[r];
    }
}

#define HGS_K7_PARAMS                                                                                                 \
    int N, const uint32_t *__restrict__ sorted_of_gid, const acc_t *__restrict__ accum, int acc_stride, int n4,     \
        const float *__restrict__ p4, int64_t cap4, const float *__restrict__ p3, int64_t cap3, int deg,           \
        DevCamera cam, double t, double scale, float *__restrict__ g4, float *__restrict__ g3,                     \
        float *__restrict__ sn4, float *__restrict__ sn3, float *__restrict__ gn4, float *__restrict__ gn3,        \
        float *__restrict__ cnt4, float *__restrict__ cnt3, const double *__restrict__ conic_src, int conic_stride, \
        const float4 *__restrict__ ddir, int first
#define HGS_K7_ARGS                                                                                              \
    N, sorted_of_gid, accum, acc_stride, n4, p4, cap4, p3, cap3, deg, cam, t, scale, g4, g3, sn4, sn3, gn4, gn3, \
        cnt4, cnt3, conic_src, conic_stride, ddir, first

__global__ void __launch_bounds__(128, 4) gaussian_bwd_kernel(HGS_K7_PARAMS) {
    pdl_wait();  // launched with launch_pdl
    gaussian_bwd_body<false>(HGS_K7_ARGS);
}

__global__ void __launch_bounds__(128) gaussian_bwd_exact_kernel(HGS_K7_PARAMS) {
    pdl_wait();  // launched with launch_pdl
    gaussian_bwd_body<true>(HGS_K7_ARGS);
}

// K7b: SH colour backward (backward.cpp:252-273), one thread per visible
// Gaussian, FP32: dL/dSH_k = scale * Y_k(dir) * dL/drgb (zero on clamped
// channels) into the SH gradient rows, and dL/d(dir) = sum_k (dL/drgb . SH_k)
// dY_k/d(dir) for K7 (which chains it into the mean).  The view direction and
// the clamped-channel mask were recorded by K1.  Split from K7 so the
// FP64 geometry kernel carries no SH state (occupancy) and the 48-row
// coefficient / gradient traffic runs at high memory-level parallelism.
__global__ void __launch_bounds__(128) sh_bwd_kernel(int N, const uint32_t* __restrict__ sorted_of_gid,
                                                     const acc_t* __restrict__ accum, int acc_stride, int n4,
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
    HGS_DCHECK(j < g_chk.splats);
    const acc_t* acc = accum + (size_t)j * acc_stride;
    const double2 a01 = *reinterpret_cast<const double2*>(acc), a23 = *reinterpret_cast<const double2*>(acc + 2),
                  a45 = *reinterpret_cast<const double2*>(acc + 4), a67 = *reinterpret_cast<const double2*>(acc + 6);
    if (a01.x == 0.0 && a01.y == 0.0 && a23.x == 0.0 && a23.y == 0.0 && a45.x == 0.0 && a45.y == 0.0 &&
        a67.x == 0.0 && a67.y == 0.0 && acc[8] == 0.0)
        return;  // untouched (backward.cpp:226): K7 skips it too
    const bool dyn = gid < n4;
    const int i = dyn ? gid : gid - n4;
    float* Gs = (dyn ? g4 : g3) + i;
    const int64_t cap = dyn ? cap4 : cap3;
    const int shrow = dyn ? R4_SH : R3_SH;
    const ShRec sr = shrec[gid];
    const float df[3] = {sr.dir.x, sr.dir.y, sr.dir.z};
    const uint32_t clamped = __float_as_uint(sr.dir.w);
    const float d_rgb[3] = {(float)a01.x, (float)a01.y, (float)a23.x};
    float drr[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) drr[c] = ((clamped >> c) & 1u) ? 0.0f : d_rgb[c];
    float basis[16];
    sh_basis_f(df, deg, basis);
    const int K = sh_count(deg);
    // dL/d(direction) = sum_c drr_c * d rgb_c / d direction (K1's Jacobian)
    ddir[gid] = make_float4(fmaf(drr[0], sr.j[0].x, fmaf(drr[1], sr.j[1].x, drr[2] * sr.j[2].x)),
                            fmaf(drr[0], sr.j[0].y, fmaf(drr[1], sr.j[1].y, drr[2] * sr.j[2].y)),
                            fmaf(drr[0], sr.j[0].z, fmaf(drr[1], sr.j[1].z, drr[2] * sr.j[2].z)), 0.f);
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
