// hgs_oracle.cpp -- CPU FP64 restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY (see hgs_oracle.h).  Every function cites the
// reference file:line it restates; paths are relative to /root/reference/proj.
//
// Arithmetic convention: every dot product / matrix product is a left-to-right
// sequential sum and the file is compiled with -ffp-contract=off, so the
// operation order is fully specified.  The CUDA product computes the
// bit-exact quantities (depth, pixel boxes, tile rects) with the same order
// using __dmul_rn/__dadd_rn, which is what makes the key/box parity exact.
#include "hgs_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace hgso {

// raster.hpp:14-19
constexpr int kTile = 16;
constexpr double kAlphaCutoff = 1.0 / 255.0;
constexpr double kTransFloor = 1e-4;
constexpr double kAlphaClamp = 0.999;
constexpr double kLowPass = 0.3;

struct DegenerateTemporal : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DegenerateRotation : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericAbort : std::runtime_error {
    using std::runtime_error::runtime_error;
};

thread_local std::string g_err;

inline int sh_count(int deg) { return (deg + 1) * (deg + 1); }
inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }  // gauss_math.hpp:83
inline double logit(double p) { return std::log(p / (1.0 - p)); }         // gauss_math.hpp:84

// ------------------------------------------------------------ small matrices
struct M3 {
    double a[3][3];
};
struct M4 {
    double a[4][4];
};

inline M3 mul3(const M3& x, const M3& y) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = x.a[i][0] * y.a[0][j];
            s = s + x.a[i][1] * y.a[1][j];
            s = s + x.a[i][2] * y.a[2][j];
            r.a[i][j] = s;
        }
    return r;
}
inline M3 mul3T(const M3& x, const M3& y) {  // x * y^T
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = x.a[i][0] * y.a[j][0];
            s = s + x.a[i][1] * y.a[j][1];
            s = s + x.a[i][2] * y.a[j][2];
            r.a[i][j] = s;
        }
    return r;
}
inline M3 tr3(const M3& x) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[j][i];
    return r;
}
inline M4 mul4(const M4& x, const M4& y) {
    M4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = x.a[i][0] * y.a[0][j];
            s = s + x.a[i][1] * y.a[1][j];
            s = s + x.a[i][2] * y.a[2][j];
            s = s + x.a[i][3] * y.a[3][j];
            r.a[i][j] = s;
        }
    return r;
}
inline double det3(const M3& m) {
    const auto& a = m.a;
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) -
           a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

// ------------------------------------------------------------ quaternions
// gauss_math.cpp:13-24
void canonicalize(double& w, double& x, double& y, double& z) {
    bool flip = false;
    if (w < 0.0) {
        flip = true;
    } else if (w == 0.0) {
        if (x != 0.0) flip = x < 0.0;
        else if (y != 0.0) flip = y < 0.0;
        else flip = z < 0.0;
    }
    if (flip) { w = -w; x = -x; y = -y; z = -z; }
}

// gauss_math.cpp:35-44 UnitQuat::normalized
void quat_normalized(double w, double x, double y, double z, double out[4]) {
    double n = std::sqrt(w * w + x * x + y * y + z * z);
    if (!(n > 0.0) || !std::isfinite(n))
        throw std::invalid_argument("UnitQuat: cannot normalize zero/non-finite quaternion");
    w /= n; x /= n; y /= n; z /= n;
    canonicalize(w, x, y, z);
    out[0] = w; out[1] = x; out[2] = y; out[3] = z;
}

inline double qnorm(const double q[4]) {
    return std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
}

// gauss_math.cpp:48-58
M3 quat_to_rot3(const double q[4]) {
    double n = qnorm(q);
    if (std::abs(n - 1.0) > 1e-6) throw std::invalid_argument("quat_to_rot3: non-unit quaternion");
    double w = q[0], x = q[1], y = q[2], z = q[3];
    M3 r;
    r.a[0][0] = 1 - 2 * (y * y + z * z);
    r.a[0][1] = 2 * (x * y - z * w);
    r.a[0][2] = 2 * (x * z + y * w);
    r.a[1][0] = 2 * (x * y + z * w);
    r.a[1][1] = 1 - 2 * (x * x + z * z);
    r.a[1][2] = 2 * (y * z - x * w);
    r.a[2][0] = 2 * (x * z - y * w);
    r.a[2][1] = 2 * (y * z + x * w);
    r.a[2][2] = 1 - 2 * (x * x + y * y);
    return r;
}

// gauss_math.cpp:60-63
bool is_rotation(const M3& m, double tol) {
    M3 p = mul3(tr3(m), m);
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            worst = std::max(worst, std::abs(p.a[i][j] - (i == j ? 1.0 : 0.0)));
    return worst <= tol && std::abs(det3(m) - 1.0) <= tol;
}

// gauss_math.cpp:70-97
void rot3_to_quat(const M3& m, double q[4]) {
    if (!is_rotation(m, 1e-6)) throw std::invalid_argument("rot3_to_quat: input is not a rotation matrix");
    const auto& r = m.a;
    double tr = r[0][0] + r[1][1] + r[2][2];
    double w, x, y, z;
    if (1.0 + tr >= 1e-6) {
        w = 0.5 * std::sqrt(1.0 + tr);
        x = (r[2][1] - r[1][2]) / (4.0 * w);
        y = (r[0][2] - r[2][0]) / (4.0 * w);
        z = (r[1][0] - r[0][1]) / (4.0 * w);
    } else {
        int i = 0;
        if (r[1][1] > r[0][0]) i = 1;
        if (r[2][2] > r[i][i]) i = 2;
        int j = (i + 1) % 3, k = (i + 2) % 3;
        double s = std::sqrt(r[i][i] - r[j][j] - r[k][k] + 1.0);
        double v[3];
        v[i] = 0.5 * s;
        double inv = 0.5 / s;
        w = (r[k][j] - r[j][k]) * inv;
        v[j] = (r[j][i] + r[i][j]) * inv;
        v[k] = (r[k][i] + r[i][k]) * inv;
        x = v[0]; y = v[1]; z = v[2];
    }
    quat_normalized(w, x, y, z, q);
}

// gauss_math.cpp:99-117
M4 left_isoclinic(const double q[4]) {
    double a = q[0], b = q[1], c = q[2], d = q[3];
    M4 m = {{{a, -b, -c, -d}, {b, a, -d, c}, {c, d, a, -b}, {d, -c, b, a}}};
    return m;
}
M4 right_isoclinic(const double q[4]) {
    double p = q[0], qq = q[1], r = q[2], s = q[3];
    M4 m = {{{p, -qq, -r, -s}, {qq, p, s, -r}, {r, -s, p, qq}, {s, r, -qq, p}}};
    return m;
}
// gauss_math.cpp:119-121
M4 rot4_from_pair(const double ql[4], const double qr[4]) {
    return mul4(left_isoclinic(ql), right_isoclinic(qr));
}

// gauss_math.cpp:154-157  Sigma = (R diag e^s)(R diag e^s)^T
M3 build_cov3(const M3& rot, const double ls[3]) {
    double e[3] = {std::exp(ls[0]), std::exp(ls[1]), std::exp(ls[2])};
    M3 m;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) m.a[i][j] = rot.a[i][j] * e[j];
    return mul3T(m, m);
}
// gauss_math.cpp:159-162
M4 build_cov4(const M4& rot, const double ls[4]) {
    double e[4] = {std::exp(ls[0]), std::exp(ls[1]), std::exp(ls[2]), std::exp(ls[3])};
    M4 m;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) m.a[i][j] = rot.a[i][j] * e[j];
    M4 r;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) {
            double s = m.a[i][0] * m.a[j][0];
            s = s + m.a[i][1] * m.a[j][1];
            s = s + m.a[i][2] * m.a[j][2];
            s = s + m.a[i][3] * m.a[j][3];
            r.a[i][j] = s;
        }
    return r;
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (stands in for
// Eigen::SelfAdjointEigenSolver<Mat3>, gauss_math.cpp:166; exact bits are
// parity-unpinned, properties are pinned by test_gauss_math.cpp:113-148).
// Eigenvalues ascending, eigenvectors in the columns of v.
void jacobi_eig3(const M3& in, double ev[3], M3& v) {
    M3 a = in;
    v = M3{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = std::abs(a.a[0][1]) + std::abs(a.a[0][2]) + std::abs(a.a[1][2]);
        double diag = std::abs(a.a[0][0]) + std::abs(a.a[1][1]) + std::abs(a.a[2][2]);
        if (off <= 1e-300 || off <= 1e-18 * diag) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double apq = a.a[p][q];
                if (apq == 0.0) continue;
                double theta = (a.a[q][q] - a.a[p][p]) / (2.0 * apq);
                double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {  // A <- J^T A J
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
    std::sort(idx, idx + 3, [&](int x, int y) { return a.a[x][x] < a.a[y][y]; });
    M3 vs;
    for (int c = 0; c < 3; ++c) {
        ev[c] = a.a[idx[c]][idx[c]];
        for (int r = 0; r < 3; ++r) vs.a[r][c] = v.a[r][idx[c]];
    }
    v = vs;
}

// gauss_math.cpp:164-173
M3 clamp_psd(const M3& m, double eps = 1e-12) {
    M3 sym;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) sym.a[i][j] = 0.5 * (m.a[i][j] + m.a[j][i]);
    double ev[3];
    M3 v;
    jacobi_eig3(sym, ev, v);
    double min_ev = std::min(ev[0], std::min(ev[1], ev[2]));
    if (min_ev >= eps) return sym;
    if (min_ev < -1e-8)
        throw std::invalid_argument("clamp_psd: matrix is indefinite beyond rounding tolerance");
    M3 vd;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) vd.a[i][j] = v.a[i][j] * std::max(ev[j], eps);
    return mul3T(vd, v);
}

struct Slice {
    double mean3[3];
    M3 cov3;
    double weight;
};

// gauss_math.cpp:175-186
Slice condition_at_time(const double mean4[4], const M4& cov4, double t) {
    double s44 = cov4.a[3][3];
    if (s44 < 1e-12) throw DegenerateTemporal("condition_at_time: temporal variance below 1e-12");
    double cross[3] = {cov4.a[0][3], cov4.a[1][3], cov4.a[2][3]};
    double dt = t - mean4[3];
    Slice s;
    double f = dt / s44;
    for (int i = 0; i < 3; ++i) s.mean3[i] = mean4[i] + cross[i] * f;
    M3 c;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) c.a[i][j] = cov4.a[i][j] - (cross[i] * cross[j]) / s44;
    s.cov3 = clamp_psd(c);
    s.weight = std::exp(-0.5 * dt * dt / s44);
    return s;
}

// One-sided (Hestenes) Jacobi SVD of a 3x3, singular values descending.
// Stands in for Eigen::JacobiSVD<Mat3> (gauss_math.cpp:190); the polar factor
// it feeds is unique, so any accurate SVD gives the same rotation.
void svd3(const M3& a, M3& u, double sv[3], M3& v) {
    M3 b = a;
    v = M3{{{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}};
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool changed = false;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                double al = 0, be = 0, ga = 0;
                for (int k = 0; k < 3; ++k) {
                    al += b.a[k][p] * b.a[k][p];
                    be += b.a[k][q] * b.a[k][q];
                    ga += b.a[k][p] * b.a[k][q];
                }
                if (ga == 0.0 || std::abs(ga) <= 1e-17 * std::sqrt(al * be)) continue;
                changed = true;
                double zeta = (be - al) / (2.0 * ga);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (int k = 0; k < 3; ++k) {
                    double bp = b.a[k][p], bq = b.a[k][q];
                    b.a[k][p] = c * bp - s * bq;
                    b.a[k][q] = s * bp + c * bq;
                    double vp = v.a[k][p], vq = v.a[k][q];
                    v.a[k][p] = c * vp - s * vq;
                    v.a[k][q] = s * vp + c * vq;
                }
            }
        if (!changed) break;
    }
    double n[3];
    for (int c = 0; c < 3; ++c)
        n[c] = std::sqrt(b.a[0][c] * b.a[0][c] + b.a[1][c] * b.a[1][c] + b.a[2][c] * b.a[2][c]);
    int idx[3] = {0, 1, 2};
    std::sort(idx, idx + 3, [&](int x, int y) { return n[x] > n[y]; });
    M3 bs, vs;
    for (int c = 0; c < 3; ++c) {
        sv[c] = n[idx[c]];
        for (int r = 0; r < 3; ++r) {
            bs.a[r][c] = b.a[r][idx[c]];
            vs.a[r][c] = v.a[r][idx[c]];
        }
    }
    v = vs;
    const double tiny = 1e-300;
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) u.a[r][c] = sv[c] > tiny ? bs.a[r][c] / sv[c] : 0.0;
    auto cross_col = [&](int c0, int c1, int dst) {
        u.a[0][dst] = u.a[1][c0] * u.a[2][c1] - u.a[2][c0] * u.a[1][c1];
        u.a[1][dst] = u.a[2][c0] * u.a[0][c1] - u.a[0][c0] * u.a[2][c1];
        u.a[2][dst] = u.a[0][c0] * u.a[1][c1] - u.a[1][c0] * u.a[0][c1];
    };
    if (sv[2] <= 1e-15 * std::max(sv[0], tiny)) cross_col(0, 1, 2);
}

// gauss_math.cpp:188-201
void extract_spatial_rot(const M4& r4, M3& rot, double& leakage) {
    M3 block;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) block.a[i][j] = r4.a[i][j];
    M3 u, v;
    double sv[3];
    svd3(block, u, sv, v);
    if (sv[0] < 1e-9) throw DegenerateRotation("extract_spatial_rot: spatial block is singular");
    M3 uvt = mul3T(u, v);
    if (det3(uvt) < 0.0)
        for (int r = 0; r < 3; ++r) u.a[r][2] = -u.a[r][2];
    rot = mul3T(u, v);
    double l2 = r4.a[0][3] * r4.a[0][3] + r4.a[1][3] * r4.a[1][3] + r4.a[2][3] * r4.a[2][3] +
                r4.a[3][0] * r4.a[3][0] + r4.a[3][1] * r4.a[3][1] + r4.a[3][2] * r4.a[3][2];
    leakage = std::sqrt(l2);
}

// ------------------------------------------------------------ SH (sh.cpp)
constexpr double C0 = 0.28209479177387814;
constexpr double C1 = 0.4886025119029199;
constexpr double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                          -1.0925484305920792, 0.5462742152960396};
constexpr double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                          0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                          -0.5900435899266435};

// sh.cpp:25-47
void sh_basis(const double dir[3], int degree, double out[16]) {
    double x = dir[0], y = dir[1], z = dir[2];
    out[0] = C0;
    if (degree < 1) return;
    out[1] = -C1 * y;
    out[2] = C1 * z;
    out[3] = -C1 * x;
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    out[4] = C2[0] * x * y;
    out[5] = C2[1] * y * z;
    out[6] = C2[2] * (2.0 * zz - xx - yy);
    out[7] = C2[3] * x * z;
    out[8] = C2[4] * (xx - yy);
    if (degree < 3) return;
    out[9] = C3[0] * y * (3.0 * xx - yy);
    out[10] = C3[1] * x * y * z;
    out[11] = C3[2] * y * (4.0 * zz - xx - yy);
    out[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = C3[4] * x * (4.0 * zz - xx - yy);
    out[14] = C3[5] * z * (xx - yy);
    out[15] = C3[6] * x * (xx - 3.0 * yy);
}

// sh.cpp:49-71 ; out[k*3 + c] = d Y_k / d dir_c
void sh_basis_grad(const double dir[3], int degree, double out[48]) {
    double x = dir[0], y = dir[1], z = dir[2];
    for (int i = 0; i < 48; ++i) out[i] = 0.0;
    auto set = [&](int k, double a, double b, double c) {
        out[k * 3 + 0] = a; out[k * 3 + 1] = b; out[k * 3 + 2] = c;
    };
    if (degree < 1) return;
    set(1, 0, -C1, 0);
    set(2, 0, 0, C1);
    set(3, -C1, 0, 0);
    if (degree < 2) return;
    double xx = x * x, yy = y * y, zz = z * z;
    set(4, C2[0] * y, C2[0] * x, 0);
    set(5, 0, C2[1] * z, C2[1] * y);
    set(6, C2[2] * (-2.0 * x), C2[2] * (-2.0 * y), C2[2] * (4.0 * z));
    set(7, C2[3] * z, 0, C2[3] * x);
    set(8, C2[4] * (2.0 * x), C2[4] * (-2.0 * y), 0);
    if (degree < 3) return;
    set(9, C3[0] * (6.0 * x * y), C3[0] * (3.0 * xx - 3.0 * yy), 0);
    set(10, C3[1] * (y * z), C3[1] * (x * z), C3[1] * (x * y));
    set(11, C3[2] * (-2.0 * x * y), C3[2] * (4.0 * zz - xx - 3.0 * yy), C3[2] * (8.0 * y * z));
    set(12, C3[3] * (-6.0 * x * z), C3[3] * (-6.0 * y * z), C3[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy));
    set(13, C3[4] * (4.0 * zz - 3.0 * xx - yy), C3[4] * (-2.0 * x * y), C3[4] * (8.0 * x * z));
    set(14, C3[5] * (2.0 * x * z), C3[5] * (-2.0 * y * z), C3[5] * (xx - yy));
    set(15, C3[6] * (3.0 * xx - 3.0 * yy), C3[6] * (-6.0 * x * y), 0);
}

// backward.cpp:44-52 (sum + 0.5, unclamped)
void sh_raw(const double* coeffs, int degree, const double dir[3], double rgb[3]) {
    double basis[16];
    sh_basis(dir, degree, basis);
    rgb[0] = rgb[1] = rgb[2] = 0.0;
    const int n = sh_count(degree);
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) rgb[c] = rgb[c] + basis[i] * coeffs[i * 3 + c];
    for (int c = 0; c < 3; ++c) rgb[c] = rgb[c] + 0.5;
}

// sh.cpp:73-83
void eval_sh(const double* coeffs, int degree, const double dir[3], double rgb[3]) {
    double n = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (std::abs(n - 1.0) > 1e-6) throw std::invalid_argument("eval_sh: view direction must be unit");
    sh_raw(coeffs, degree, dir, rgb);
    for (int c = 0; c < 3; ++c) rgb[c] = std::min(std::max(rgb[c], 0.0), 1.0);
}

// ------------------------------------------------------------ camera
struct Cam {
    double fx, fy, cx, cy;
    M3 rot;
    double trans[3];
    int width, height;
    double near_, far_;
};

Cam to_cam(const hgso_camera& c) {
    Cam k;
    k.fx = c.fx; k.fy = c.fy; k.cx = c.cx; k.cy = c.cy;
    for (int i = 0; i < 9; ++i) k.rot.a[i / 3][i % 3] = c.rot[i];
    for (int i = 0; i < 3; ++i) k.trans[i] = c.trans[i];
    k.width = c.width; k.height = c.height; k.near_ = c.near_; k.far_ = c.far_;
    return k;
}

// camera.hpp:21-26
void validate(const Cam& c) {
    if (!(c.fx > 0.0 && c.fy > 0.0)) throw std::invalid_argument("Camera: fx, fy must be positive");
    if (!(0.0 < c.near_ && c.near_ < c.far_)) throw std::invalid_argument("Camera: need 0 < near < far");
    if (c.width <= 0 || c.height <= 0) throw std::invalid_argument("Camera: bad image dimensions");
    if (!is_rotation(c.rot, 1e-8)) throw std::invalid_argument("Camera: rotation not orthonormal");
}

// camera.hpp:18  x_cam = R x + t
void to_camera(const Cam& c, const double p[3], double out[3]) {
    for (int i = 0; i < 3; ++i) {
        double s = c.rot.a[i][0] * p[0];
        s = s + c.rot.a[i][1] * p[1];
        s = s + c.rot.a[i][2] * p[2];
        out[i] = s + c.trans[i];
    }
}
// camera.hpp:19  -R^T t
void cam_position(const Cam& c, double out[3]) {
    for (int i = 0; i < 3; ++i) {
        double s = (-c.rot.a[0][i]) * c.trans[0];
        s = s + (-c.rot.a[1][i]) * c.trans[1];
        s = s + (-c.rot.a[2][i]) * c.trans[2];
        out[i] = s;
    }
}

// camera.cpp:6-22
Cam look_at(const double eye[3], const double target[3], const double up[3], double focal, int w, int h) {
    auto normalized = [](double v[3]) {
        double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        for (int i = 0; i < 3; ++i) v[i] /= n;
    };
    auto cross = [](const double a[3], const double b[3], double o[3]) {
        o[0] = a[1] * b[2] - a[2] * b[1];
        o[1] = a[2] * b[0] - a[0] * b[2];
        o[2] = a[0] * b[1] - a[1] * b[0];
    };
    double fwd[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
    normalized(fwd);
    double right[3];
    cross(fwd, up, right);
    normalized(right);
    double down[3];
    cross(fwd, right, down);
    Cam cam;
    for (int j = 0; j < 3; ++j) {
        cam.rot.a[0][j] = right[j];
        cam.rot.a[1][j] = down[j];
        cam.rot.a[2][j] = fwd[j];
    }
    for (int i = 0; i < 3; ++i) {
        double s = (-cam.rot.a[i][0]) * eye[0];
        s = s + (-cam.rot.a[i][1]) * eye[1];
        s = s + (-cam.rot.a[i][2]) * eye[2];
        cam.trans[i] = s;
    }
    cam.fx = cam.fy = focal;
    cam.cx = w / 2.0;
    cam.cy = h / 2.0;
    cam.width = w;
    cam.height = h;
    cam.near_ = 0.01;
    cam.far_ = 100.0;
    return cam;
}

hgso_camera from_cam(const Cam& k) {
    hgso_camera c;
    c.fx = k.fx; c.fy = k.fy; c.cx = k.cx; c.cy = k.cy;
    for (int i = 0; i < 9; ++i) c.rot[i] = k.rot.a[i / 3][i % 3];
    for (int i = 0; i < 3; ++i) c.trans[i] = k.trans[i];
    c.width = k.width; c.height = k.height; c.near_ = k.near_; c.far_ = k.far_;
    return c;
}

// ------------------------------------------------------------ scene access
struct View {
    const hgso_scene* s;
    int K;  // SH coefficient count
    int64_t n4() const { return s->n4; }
    int64_t n3() const { return s->n3; }
    void mean4(int64_t i, double m[4]) const {
        m[0] = s->mean_x[i * 3]; m[1] = s->mean_x[i * 3 + 1]; m[2] = s->mean_x[i * 3 + 2];
        m[3] = s->mean_t[i];
    }
    M4 rot4(int64_t i) const { return rot4_from_pair(&s->ql[i * 4], &s->qr[i * 4]); }
    M4 cov4(int64_t i) const { return build_cov4(rot4(i), &s->log_s4[i * 4]); }
    M3 cov3(int64_t i) const { return build_cov3(quat_to_rot3(&s->quat3[i * 4]), &s->log_s3[i * 3]); }
    const double* sh4(int64_t i) const { return &s->sh4[i * K * 3]; }
    const double* sh3(int64_t i) const { return &s->sh3[i * K * 3]; }
};

// ------------------------------------------------------------ projection
struct Splat {
    double sx, sy;
    double conic[2][2];
    double depth;
    double rgb[3];
    double alpha;
    int radius;
    int pool;
    uint32_t index;
};

struct Bounds {
    int x0, x1, y0, y1;
    bool empty() const { return x0 > x1 || y0 > y1; }
};

// raster.cpp:15-24
Bounds splat_bounds(const Splat& s, int w, int h) {
    int mx = int(std::floor(s.sx));
    int my = int(std::floor(s.sy));
    Bounds b;
    b.x0 = std::max(0, mx - s.radius);
    b.x1 = std::min(w - 1, mx + s.radius);
    b.y0 = std::max(0, my - s.radius);
    b.y1 = std::min(h - 1, my + s.radius);
    return b;
}

struct Jac {
    double j[2][3];
    double t[2][3];  // J * W
};

Jac make_jac(const Cam& cam, const double p[3]) {
    double z = p[2];
    Jac J;
    J.j[0][0] = cam.fx / z;
    J.j[0][1] = 0.0;
    J.j[0][2] = -cam.fx * p[0] / (z * z);
    J.j[1][0] = 0.0;
    J.j[1][1] = cam.fy / z;
    J.j[1][2] = -cam.fy * p[1] / (z * z);
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) {
            double s = J.j[i][0] * cam.rot.a[0][k];
            s = s + J.j[i][1] * cam.rot.a[1][k];
            s = s + J.j[i][2] * cam.rot.a[2][k];
            J.t[i][k] = s;
        }
    return J;
}

// raster.cpp:26-64
bool project_3d(const double mean3[3], const M3& cov3, const Cam& cam, hgso_stats* st, Splat& s) {
    double p[3];
    to_camera(cam, mean3, p);
    double z = p[2];
    if (z < cam.near_ || z > cam.far_) {
        if (st) st->culled_depth++;
        return false;
    }
    s.depth = z;
    s.sx = cam.fx * p[0] / z + cam.cx;
    s.sy = cam.fy * p[1] / z + cam.cy;
    Jac J = make_jac(cam, p);
    double tc[2][3];  // T * cov3
    for (int i = 0; i < 2; ++i)
        for (int k = 0; k < 3; ++k) {
            double a = J.t[i][0] * cov3.a[0][k];
            a = a + J.t[i][1] * cov3.a[1][k];
            a = a + J.t[i][2] * cov3.a[2][k];
            tc[i][k] = a;
        }
    double c2[2][2];
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) {
            double a = tc[i][0] * J.t[j][0];
            a = a + tc[i][1] * J.t[j][1];
            a = a + tc[i][2] * J.t[j][2];
            c2[i][j] = a;
        }
    c2[0][0] += kLowPass;
    c2[1][1] += kLowPass;
    double det = c2[0][0] * c2[1][1] - c2[0][1] * c2[1][0];
    if (det <= 1e-12) {
        if (st) st->culled_degenerate++;
        return false;
    }
    s.conic[0][0] = c2[1][1] / det;
    s.conic[0][1] = -c2[0][1] / det;
    s.conic[1][0] = -c2[1][0] / det;
    s.conic[1][1] = c2[0][0] / det;
    double mid = 0.5 * (c2[0][0] + c2[1][1]);
    double max_ev = mid + std::sqrt(std::max(0.0, mid * mid - det));
    s.radius = int(std::ceil(3.0 * std::sqrt(max_ev)));
    Bounds b = splat_bounds(s, cam.width, cam.height);
    if (b.empty()) {
        if (st) st->culled_offscreen++;
        return false;
    }
    if (st) st->projected++;
    return true;
}

void view_dir_of(const double mean3[3], const double campos[3], double dir[3], double* dist) {
    double v[3] = {mean3[0] - campos[0], mean3[1] - campos[1], mean3[2] - campos[2]};
    double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    if (dist) *dist = n;
    if (n > 0.0) {
        for (int i = 0; i < 3; ++i) dir[i] = v[i] / n;
    } else {
        dir[0] = 0; dir[1] = 0; dir[2] = 1;
    }
}

// raster.cpp:66-88
bool slice_project_4d(const View& v, int64_t i, double t, const Cam& cam, double cutoff,
                      hgso_stats* st, Splat& s, Slice* slice_out = nullptr) {
    Slice sl;
    double m4[4];
    v.mean4(i, m4);
    try {
        sl = condition_at_time(m4, v.cov4(i), t);
    } catch (const DegenerateTemporal&) {
        if (st) st->degenerate_temporal++;
        return false;
    }
    if (sl.weight < cutoff) {
        if (st) st->culled_temporal++;
        return false;
    }
    if (!project_3d(sl.mean3, sl.cov3, cam, st, s)) return false;
    s.alpha = std::min(sigmoid(v.s->op4[i]) * sl.weight, kAlphaClamp);
    double cp[3], dir[3];
    cam_position(cam, cp);
    view_dir_of(sl.mean3, cp, dir, nullptr);
    eval_sh(v.sh4(i), v.s->sh_degree, dir, s.rgb);
    s.pool = 1;
    if (slice_out) *slice_out = sl;
    return true;
}

// raster.cpp:90-116
std::vector<Splat> project_scene(const View& v, const Cam& cam, double t, double cutoff,
                                 hgso_stats* st) {
    std::vector<Splat> prims;
    prims.reserve(size_t(v.n4() + v.n3()));
    for (int64_t i = 0; i < v.n4(); ++i) {
        Splat s;
        if (slice_project_4d(v, i, t, cam, cutoff, st, s)) {
            s.index = uint32_t(i);
            prims.push_back(s);
        }
    }
    double cp[3];
    cam_position(cam, cp);
    for (int64_t i = 0; i < v.n3(); ++i) {
        Splat s;
        if (project_3d(&v.s->mean3[i * 3], v.cov3(i), cam, st, s)) {
            s.alpha = std::min(sigmoid(v.s->op3[i]), kAlphaClamp);
            double dir[3];
            view_dir_of(&v.s->mean3[i * 3], cp, dir, nullptr);
            eval_sh(v.sh3(i), v.s->sh_degree, dir, s.rgb);
            s.pool = 0;
            s.index = uint32_t(i);
            prims.push_back(s);
        }
    }
    return prims;
}

uint32_t f32_bits(double d) {
    float f = float(d);
    uint32_t b;
    std::memcpy(&b, &f, 4);
    return b;
}

// raster.cpp:123-148
template <typename It>
void composite_pixel(int px, int py, It begin, It end, const std::vector<Splat>& prims,
                     const double bg[3], int w, int h, double out[3], uint32_t* out_count,
                     double* out_trans, std::vector<uint32_t>* contribs = nullptr) {
    double trans = 1.0;
    double acc[3] = {0, 0, 0};
    uint32_t count = 0;
    double pc[2] = {px + 0.5, py + 0.5};
    for (It it = begin; it != end; ++it) {
        const Splat& s = prims[*it];
        Bounds b = splat_bounds(s, w, h);
        if (px < b.x0 || px > b.x1 || py < b.y0 || py > b.y1) continue;
        if (out_count) count++;
        double d0 = pc[0] - s.sx, d1 = pc[1] - s.sy;
        double q0 = s.conic[0][0] * d0 + s.conic[0][1] * d1;
        double q1 = s.conic[1][0] * d0 + s.conic[1][1] * d1;
        double power = 0.5 * (d0 * q0 + d1 * q1);
        double a = s.alpha * std::exp(-power);
        if (a < kAlphaCutoff) continue;
        for (int c = 0; c < 3; ++c) acc[c] = acc[c] + s.rgb[c] * (a * trans);
        if (contribs) contribs->push_back(*it);
        trans *= 1.0 - a;
        if (trans < kTransFloor) break;
    }
    for (int c = 0; c < 3; ++c) out[c] = acc[c] + trans * bg[c];
    if (out_count) *out_count = count;
    if (out_trans) *out_trans = trans;
}

// raster.cpp:150-163
void run_tiles(int tile_count, int num_threads, const std::function<void(int)>& work) {
    if (num_threads <= 1) {
        for (int i = 0; i < tile_count; ++i) work(i);
        return;
    }
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < num_threads; ++t)
        pool.emplace_back([&] {
            for (int i = next.fetch_add(1); i < tile_count; i = next.fetch_add(1)) work(i);
        });
    for (auto& th : pool) th.join();
}

struct Instance {
    uint64_t key;
    uint32_t prim;
    bool operator<(const Instance& o) const { return key != o.key ? key < o.key : prim < o.prim; }
};

// raster.cpp:180-212 : duplication, sort, ranges
void build_instances(const std::vector<Splat>& prims, const Cam& cam, std::vector<Instance>& inst,
                     std::vector<std::pair<size_t, size_t>>& ranges, int& tiles_x) {
    tiles_x = (cam.width + kTile - 1) / kTile;
    const int tiles_y = (cam.height + kTile - 1) / kTile;
    const int tile_count = tiles_x * tiles_y;
    inst.clear();
    for (uint32_t i = 0; i < prims.size(); ++i) {
        Bounds b = splat_bounds(prims[i], cam.width, cam.height);
        if (b.empty()) continue;
        uint32_t db = f32_bits(prims[i].depth);
        for (int ty = b.y0 / kTile; ty <= b.y1 / kTile; ++ty)
            for (int tx = b.x0 / kTile; tx <= b.x1 / kTile; ++tx) {
                uint64_t tile_id = uint64_t(ty) * tiles_x + tx;
                inst.push_back({(tile_id << 32) | db, i});
            }
    }
    std::sort(inst.begin(), inst.end());
    ranges.assign(size_t(tile_count), {0, 0});
    for (size_t i = 0; i < inst.size();) {
        uint64_t tile_id = inst[i].key >> 32;
        size_t j = i;
        while (j < inst.size() && (inst[j].key >> 32) == tile_id) ++j;
        ranges[size_t(tile_id)] = {i, j};
        i = j;
    }
}

// raster.cpp:167-235
void rasterize(const View& v, const Cam& cam, double t, const double bg[3], double cutoff,
               int num_threads, double* rgb, uint32_t* counts, double* trans, hgso_stats* st,
               std::vector<Splat>* prims_out = nullptr,
               std::vector<std::vector<uint32_t>>* contribs = nullptr) {
    validate(cam);
    hgso_stats local{};
    std::vector<Splat> prims = project_scene(v, cam, t, cutoff, &local);
    if (st) *st = local;
    std::vector<Instance> inst;
    std::vector<std::pair<size_t, size_t>> ranges;
    int tiles_x;
    build_instances(prims, cam, inst, ranges, tiles_x);
    const int W = cam.width, H = cam.height;
    run_tiles(int(ranges.size()), num_threads, [&](int tile) {
        auto [lo, hi] = ranges[size_t(tile)];
        int tx = tile % tiles_x, ty = tile / tiles_x;
        int x0 = tx * kTile, y0 = ty * kTile;
        int x1 = std::min(W, x0 + kTile), y1 = std::min(H, y0 + kTile);
        std::vector<uint32_t> order;
        order.reserve(hi - lo);
        for (size_t i = lo; i < hi; ++i) order.push_back(inst[i].prim);
        for (int py = y0; py < y1; ++py)
            for (int px = x0; px < x1; ++px) {
                size_t pix = size_t(py) * W + px;
                double out[3];
                composite_pixel(px, py, order.begin(), order.end(), prims, bg, W, H, out,
                                counts ? &counts[pix] : nullptr, trans ? &trans[pix] : nullptr,
                                contribs ? &(*contribs)[pix] : nullptr);
                for (int c = 0; c < 3; ++c) rgb[pix * 3 + c] = out[c];
            }
    });
    if (prims_out) *prims_out = std::move(prims);
}

// raster.cpp:237-266
void reference_render(const View& v, const Cam& cam, double t, const double bg[3], double cutoff,
                      double* rgb, hgso_stats* st) {
    validate(cam);
    hgso_stats local{};
    std::vector<Splat> prims = project_scene(v, cam, t, cutoff, &local);
    if (st) *st = local;
    std::vector<uint32_t> order(prims.size());
    for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        float da = float(prims[a].depth), db = float(prims[b].depth);
        return da != db ? da < db : a < b;
    });
    for (int py = 0; py < cam.height; ++py)
        for (int px = 0; px < cam.width; ++px) {
            size_t pix = size_t(py) * cam.width + px;
            double out[3];
            composite_pixel(px, py, order.begin(), order.end(), prims, bg, cam.width, cam.height,
                            out, nullptr, nullptr);
            for (int c = 0; c < 3; ++c) rgb[pix * 3 + c] = out[c];
        }
}

// ------------------------------------------------------------ taped forward
// backward.hpp:42-65
struct PrimTape {
    Splat splat;
    double cam_p[3];
    M3 cov3;
    double mean3[3];
    double weight = 1.0;
    double raw_rgb[3];
    double view_dir[3];
    double view_dist = 0.0;
    bool alpha_clamped = false;
    M4 cov4;
    M4 rot4;
};

struct Tape {
    std::vector<PrimTape> prims;
    std::vector<std::vector<uint32_t>> contribs;
    std::vector<double> final_trans;
    double bg[3];
    double time = 0.0;
    int width = 0, height = 0;
};

// backward.cpp:89-140 : per-primitive tape records, dynamics then statics.
std::vector<PrimTape> tape_prims(const View& v, const Cam& cam, double t, double cutoff) {
    std::vector<PrimTape> out;
    double cp[3];
    cam_position(cam, cp);
    for (int64_t i = 0; i < v.n4(); ++i) {
        Splat s;
        Slice sl;
        if (!slice_project_4d(v, i, t, cam, cutoff, nullptr, s, &sl)) continue;
        s.index = uint32_t(i);
        PrimTape pt;
        pt.cov4 = v.cov4(i);
        pt.rot4 = v.rot4(i);
        for (int k = 0; k < 3; ++k) pt.mean3[k] = sl.mean3[k];
        pt.cov3 = sl.cov3;
        pt.weight = sl.weight;
        to_camera(cam, sl.mean3, pt.cam_p);
        view_dir_of(sl.mean3, cp, pt.view_dir, &pt.view_dist);
        sh_raw(v.sh4(i), v.s->sh_degree, pt.view_dir, pt.raw_rgb);
        pt.alpha_clamped = sigmoid(v.s->op4[i]) * sl.weight >= kAlphaClamp;
        pt.splat = s;
        out.push_back(pt);
    }
    for (int64_t i = 0; i < v.n3(); ++i) {
        M3 cov3 = v.cov3(i);
        Splat s;
        const double* m = &v.s->mean3[i * 3];
        if (!project_3d(m, cov3, cam, nullptr, s)) continue;
        s.alpha = std::min(sigmoid(v.s->op3[i]), kAlphaClamp);
        s.pool = 0;
        s.index = uint32_t(i);
        PrimTape pt;
        for (int k = 0; k < 3; ++k) pt.mean3[k] = m[k];
        pt.cov3 = cov3;
        to_camera(cam, m, pt.cam_p);
        view_dir_of(m, cp, pt.view_dir, &pt.view_dist);
        sh_raw(v.sh3(i), v.s->sh_degree, pt.view_dir, pt.raw_rgb);
        pt.alpha_clamped = sigmoid(v.s->op3[i]) >= kAlphaClamp;
        for (int c = 0; c < 3; ++c) s.rgb[c] = std::min(std::max(pt.raw_rgb[c], 0.0), 1.0);
        pt.splat = s;
        out.push_back(pt);
    }
    return out;
}

// Tiled forward with the tape.  Its image is bitwise identical to both
// rasterize() and the literal untiled forward_train (backward.cpp:142-175):
// a pixel's tile list is exactly the set of splats whose clamped box can
// cover it, in the same (f32 depth, projected index) order.
Tape* forward_train_tiled(const View& v, const Cam& cam, double t, const double bg[3], double cutoff,
                          int num_threads, double* rgb) {
    validate(cam);
    Tape* tape = new Tape();
    for (int c = 0; c < 3; ++c) tape->bg[c] = bg[c];
    tape->time = t;
    tape->width = cam.width;
    tape->height = cam.height;
    tape->prims = tape_prims(v, cam, t, cutoff);
    std::vector<Splat> prims(tape->prims.size());
    for (size_t i = 0; i < prims.size(); ++i) prims[i] = tape->prims[i].splat;
    size_t npx = size_t(cam.width) * cam.height;
    tape->contribs.assign(npx, {});
    tape->final_trans.assign(npx, 1.0);
    std::vector<Instance> inst;
    std::vector<std::pair<size_t, size_t>> ranges;
    int tiles_x;
    build_instances(prims, cam, inst, ranges, tiles_x);
    const int W = cam.width, H = cam.height;
    run_tiles(int(ranges.size()), num_threads, [&](int tile) {
        auto [lo, hi] = ranges[size_t(tile)];
        int tx = tile % tiles_x, ty = tile / tiles_x;
        int x0 = tx * kTile, y0 = ty * kTile;
        int x1 = std::min(W, x0 + kTile), y1 = std::min(H, y0 + kTile);
        std::vector<uint32_t> order;
        for (size_t i = lo; i < hi; ++i) order.push_back(inst[i].prim);
        for (int py = y0; py < y1; ++py)
            for (int px = x0; px < x1; ++px) {
                size_t pix = size_t(py) * W + px;
                double out[3];
                composite_pixel(px, py, order.begin(), order.end(), prims, bg, W, H, out, nullptr,
                                &tape->final_trans[pix], &tape->contribs[pix]);
                for (int c = 0; c < 3; ++c) rgb[pix * 3 + c] = out[c];
            }
    });
    return tape;
}

// backward.cpp:89-176, literally (global depth sort, every prim per pixel).
Tape* forward_train_untiled(const View& v, const Cam& cam, double t, const double bg[3], double cutoff,
                            double* rgb) {
    validate(cam);
    Tape* tape = new Tape();
    for (int c = 0; c < 3; ++c) tape->bg[c] = bg[c];
    tape->time = t;
    tape->width = cam.width;
    tape->height = cam.height;
    tape->prims = tape_prims(v, cam, t, cutoff);
    std::vector<uint32_t> order(tape->prims.size());
    for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        float da = float(tape->prims[a].splat.depth), db = float(tape->prims[b].splat.depth);
        return da != db ? da < db : a < b;
    });
    size_t npx = size_t(cam.width) * cam.height;
    tape->contribs.assign(npx, {});
    tape->final_trans.assign(npx, 1.0);
    for (int py = 0; py < cam.height; ++py)
        for (int px = 0; px < cam.width; ++px) {
            size_t pix = size_t(py) * cam.width + px;
            double trans = 1.0;
            double acc[3] = {0, 0, 0};
            double pc[2] = {px + 0.5, py + 0.5};
            for (uint32_t oi : order) {
                const Splat& s = tape->prims[oi].splat;
                Bounds b = splat_bounds(s, cam.width, cam.height);
                if (px < b.x0 || px > b.x1 || py < b.y0 || py > b.y1) continue;
                double d0 = pc[0] - s.sx, d1 = pc[1] - s.sy;
                double q0 = s.conic[0][0] * d0 + s.conic[0][1] * d1;
                double q1 = s.conic[1][0] * d0 + s.conic[1][1] * d1;
                double a = s.alpha * std::exp(-0.5 * (d0 * q0 + d1 * q1));
                if (a < kAlphaCutoff) continue;
                for (int c = 0; c < 3; ++c) acc[c] = acc[c] + s.rgb[c] * (a * trans);
                tape->contribs[pix].push_back(oi);
                trans *= 1.0 - a;
                if (trans < kTransFloor) break;
            }
            for (int c = 0; c < 3; ++c) acc[c] = acc[c] + trans * bg[c];
            tape->final_trans[pix] = trans;
            for (int c = 0; c < 3; ++c) rgb[pix * 3 + c] = acc[c];
        }
    return tape;
}

// ------------------------------------------------------------ backward
// backward.cpp:54-72
M3 drot3_dq(const double q[4], int k) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    M3 d;
    switch (k) {
        case 0: d = M3{{{0, -z, y}, {z, 0, -x}, {-y, x, 0}}}; break;
        case 1: d = M3{{{0, y, z}, {y, -2 * x, -w}, {z, w, -2 * x}}}; break;
        case 2: d = M3{{{-2 * y, x, w}, {x, 0, z}, {-w, z, -2 * y}}}; break;
        default: d = M3{{{-2 * z, -w, x}, {w, -2 * z, y}, {x, y, 0}}}; break;
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) d.a[i][j] *= 2.0;
    return d;
}

// backward.cpp:74-76
void through_normalization(const double q[4], const double g[4], double out[4]) {
    double dot = q[0] * g[0] + q[1] * g[1] + q[2] * g[2] + q[3] * g[3];
    for (int k = 0; k < 4; ++k) out[k] = g[k] - dot * q[k];
}

struct PrimAccum {
    double d_rgb[3] = {0, 0, 0};
    double d_alpha = 0.0;
    double d_screen[2] = {0, 0};
    double d_conic[2][2] = {{0, 0}, {0, 0}};
    bool touched = false;
};

// backward.cpp:178-356
void backward(const View& v, const Cam& cam, const Tape& tape, const double* lg, hgso_grads& G) {
    std::vector<PrimAccum> accum(tape.prims.size());
    for (int py = 0; py < tape.height; ++py)
        for (int px = 0; px < tape.width; ++px) {
            size_t pix = size_t(py) * tape.width + px;
            const auto& list = tape.contribs[pix];
            if (list.empty()) continue;
            double gp[3] = {lg[pix * 3], lg[pix * 3 + 1], lg[pix * 3 + 2]};
            // gpix.isZero() (backward.cpp:189): Eigen's isZero is every
            // |component| <= dummy_precision = 1e-12, not == 0
            if (std::abs(gp[0]) <= 1e-12 && std::abs(gp[1]) <= 1e-12 && std::abs(gp[2]) <= 1e-12) continue;
            double pc[2] = {px + 0.5, py + 0.5};
            const size_t n = list.size();
            std::vector<double> av(n), tv(n), gv(n);
            double trans = 1.0;
            for (size_t i = 0; i < n; ++i) {
                const Splat& s = tape.prims[list[i]].splat;
                double d0 = pc[0] - s.sx, d1 = pc[1] - s.sy;
                double q0 = s.conic[0][0] * d0 + s.conic[0][1] * d1;
                double q1 = s.conic[1][0] * d0 + s.conic[1][1] * d1;
                gv[i] = std::exp(-0.5 * (d0 * q0 + d1 * q1));
                av[i] = s.alpha * gv[i];
                tv[i] = trans;
                trans *= 1.0 - av[i];
            }
            double suffix[3] = {trans * tape.bg[0], trans * tape.bg[1], trans * tape.bg[2]};
            for (size_t ri = n; ri-- > 0;) {
                const uint32_t prim = list[ri];
                const Splat& s = tape.prims[prim].splat;
                PrimAccum& acc = accum[prim];
                acc.touched = true;
                double a = av[ri], g = gv[ri], ti = tv[ri];
                for (int c = 0; c < 3; ++c) acc.d_rgb[c] += (a * ti) * gp[c];
                double d_a = 0.0;
                for (int c = 0; c < 3; ++c) d_a += gp[c] * (s.rgb[c] * ti - suffix[c] / (1.0 - a));
                for (int c = 0; c < 3; ++c) suffix[c] += s.rgb[c] * (a * ti);
                acc.d_alpha += g * d_a;
                double d_g = s.alpha * d_a;
                double d0 = pc[0] - s.sx, d1 = pc[1] - s.sy;
                double q0 = s.conic[0][0] * d0 + s.conic[0][1] * d1;
                double q1 = s.conic[1][0] * d0 + s.conic[1][1] * d1;
                acc.d_screen[0] += (g * d_g) * q0;
                acc.d_screen[1] += (g * d_g) * q1;
                double f = -0.5 * g * d_g;
                acc.d_conic[0][0] += f * (d0 * d0);
                acc.d_conic[0][1] += f * (d0 * d1);
                acc.d_conic[1][0] += f * (d1 * d0);
                acc.d_conic[1][1] += f * (d1 * d1);
            }
        }

    double campos[3];
    cam_position(cam, campos);
    const int deg = v.s->sh_degree;
    const int n_sh = sh_count(deg);
    for (size_t pi = 0; pi < tape.prims.size(); ++pi) {
        if (!accum[pi].touched) continue;
        const PrimTape& pt = tape.prims[pi];
        const PrimAccum& acc = accum[pi];
        const Splat& s = pt.splat;
        // conic = inverse(cov2): d_cov2 = -C dC C
        double cd[2][2], d_cov2[2][2];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) cd[i][j] = s.conic[i][0] * acc.d_conic[0][j] + s.conic[i][1] * acc.d_conic[1][j];
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j) d_cov2[i][j] = -(cd[i][0] * s.conic[0][j] + cd[i][1] * s.conic[1][j]);
        double z = pt.cam_p[2], xq = pt.cam_p[0], yq = pt.cam_p[1];
        Jac J = make_jac(cam, pt.cam_p);
        // d_cov3 = T^T d_cov2 T
        double dt_[2][3];  // d_cov2 * T
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k) dt_[i][k] = d_cov2[i][0] * J.t[0][k] + d_cov2[i][1] * J.t[1][k];
        M3 d_cov3;
        for (int i = 0; i < 3; ++i)
            for (int k = 0; k < 3; ++k) d_cov3.a[i][k] = J.t[0][i] * dt_[0][k] + J.t[1][i] * dt_[1][k];
        // d_tmat = 2 d_cov2 T cov3
        double d_tmat[2][3];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k) {
                double a = 0.0;
                for (int m = 0; m < 3; ++m) a += dt_[i][m] * pt.cov3.a[m][k];
                d_tmat[i][k] = 2.0 * a;
            }
        // d_jac = d_tmat * W^T
        double d_jac[2][3];
        for (int i = 0; i < 2; ++i)
            for (int k = 0; k < 3; ++k) {
                double a = 0.0;
                for (int m = 0; m < 3; ++m) a += d_tmat[i][m] * cam.rot.a[k][m];
                d_jac[i][k] = a;
            }
        double d_cam_p[3];
        for (int k = 0; k < 3; ++k) d_cam_p[k] = J.j[0][k] * acc.d_screen[0] + J.j[1][k] * acc.d_screen[1];
        double fx = cam.fx, fy = cam.fy;
        d_cam_p[0] += d_jac[0][2] * (-fx / (z * z));
        d_cam_p[1] += d_jac[1][2] * (-fy / (z * z));
        d_cam_p[2] += d_jac[0][0] * (-fx / (z * z)) + d_jac[1][1] * (-fy / (z * z)) +
                      d_jac[0][2] * (2.0 * fx * xq / (z * z * z)) +
                      d_jac[1][2] * (2.0 * fy * yq / (z * z * z));
        double d_mean3[3];
        for (int k = 0; k < 3; ++k)
            d_mean3[k] = cam.rot.a[0][k] * d_cam_p[0] + cam.rot.a[1][k] * d_cam_p[1] + cam.rot.a[2][k] * d_cam_p[2];

        // colour path (backward.cpp:252-273)
        double d_rgb_raw[3];
        for (int c = 0; c < 3; ++c)
            d_rgb_raw[c] = (pt.raw_rgb[c] < 0.0 || pt.raw_rgb[c] > 1.0) ? 0.0 : acc.d_rgb[c];
        double basis[16], bgrad[48];
        sh_basis(pt.view_dir, deg, basis);
        sh_basis_grad(pt.view_dir, deg, bgrad);
        const double* coeffs = s.pool == 0 ? v.sh3(s.index) : v.sh4(s.index);
        double d_dir[3] = {0, 0, 0};
        double d_sh[48];
        for (int k = 0; k < n_sh; ++k) {
            double dotc = 0.0;
            for (int c = 0; c < 3; ++c) {
                d_sh[k * 3 + c] = basis[k] * d_rgb_raw[c];
                dotc += d_rgb_raw[c] * coeffs[k * 3 + c];
            }
            for (int c = 0; c < 3; ++c) d_dir[c] += bgrad[k * 3 + c] * dotc;
        }
        if (pt.view_dist > 0.0) {
            for (int i = 0; i < 3; ++i) {
                double a = 0.0;
                for (int j = 0; j < 3; ++j) {
                    double jn = ((i == j ? 1.0 : 0.0) - pt.view_dir[i] * pt.view_dir[j]) / pt.view_dist;
                    a += jn * d_dir[j];
                }
                d_mean3[i] += a;
            }
        }
        double screen_norm = std::sqrt(acc.d_screen[0] * acc.d_screen[0] + acc.d_screen[1] * acc.d_screen[1]);
        M3 d_cov3_sym;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) d_cov3_sym.a[i][j] = 0.5 * (d_cov3.a[i][j] + d_cov3.a[j][i]);

        if (s.pool == 0) {
            const int64_t i = s.index;
            for (int k = 0; k < 3; ++k) G.mean3[i * 3 + k] += d_mean3[k];
            G.screen_norm3[i] += screen_norm;
            for (int k = 0; k < n_sh * 3; ++k) G.sh3[i * n_sh * 3 + k] += d_sh[k];
            if (!pt.alpha_clamped) {
                double sg = sigmoid(v.s->op3[i]);
                G.op3[i] += acc.d_alpha * sg * (1.0 - sg);
            }
            const double* q = &v.s->quat3[i * 4];
            M3 rot = quat_to_rot3(q);
            const double* ls = &v.s->log_s3[i * 3];
            double es[3] = {std::exp(ls[0]), std::exp(ls[1]), std::exp(ls[2])};
            M3 m;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) m.a[a][b] = rot.a[a][b] * es[b];
            M3 d_m = mul3(d_cov3_sym, m);
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) d_m.a[a][b] *= 2.0;
            for (int k = 0; k < 3; ++k) {
                double a = 0.0;
                for (int r = 0; r < 3; ++r) a += d_m.a[r][k] * m.a[r][k];
                G.log_s3[i * 3 + k] += a;
            }
            M3 d_rot;
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) d_rot.a[a][b] = d_m.a[a][b] * es[b];
            double dq[4];
            for (int k = 0; k < 4; ++k) {
                M3 dr = drot3_dq(q, k);
                double a = 0.0;
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) a += d_rot.a[r][c] * dr.a[r][c];
                dq[k] = a;
            }
            double tn[4];
            through_normalization(q, dq, tn);
            for (int k = 0; k < 4; ++k) G.quat3[i * 4 + k] += tn[k];
        } else {
            const int64_t i = s.index;
            G.screen_norm4[i] += screen_norm;
            for (int k = 0; k < n_sh * 3; ++k) G.sh4[i * n_sh * 3 + k] += d_sh[k];
            double d_weight = 0.0;
            double sg = sigmoid(v.s->op4[i]);
            if (!pt.alpha_clamped) {
                G.op4[i] += acc.d_alpha * pt.weight * sg * (1.0 - sg);
                d_weight += acc.d_alpha * sg;
            }
            double s44 = pt.cov4.a[3][3];
            double cross[3] = {pt.cov4.a[0][3], pt.cov4.a[1][3], pt.cov4.a[2][3]};
            double dt = tape.time - v.s->mean_t[i];
            const double* dms = d_mean3;
            for (int k = 0; k < 3; ++k) G.mean_x[i * 3 + k] += dms[k];
            double dmc = dms[0] * cross[0] + dms[1] * cross[1] + dms[2] * cross[2];
            G.mean_t[i] += -dmc / s44 + d_weight * pt.weight * dt / s44;
            double sc[3];  // d_cov3_sym * cross
            for (int a = 0; a < 3; ++a)
                sc[a] = d_cov3_sym.a[a][0] * cross[0] + d_cov3_sym.a[a][1] * cross[1] + d_cov3_sym.a[a][2] * cross[2];
            double d_cross[3];
            for (int a = 0; a < 3; ++a) d_cross[a] = dms[a] * (dt / s44) - 2.0 * sc[a] / s44;
            double csc = cross[0] * sc[0] + cross[1] * sc[1] + cross[2] * sc[2];
            double d_s44 = -dmc * dt / (s44 * s44) + csc / (s44 * s44) +
                           d_weight * pt.weight * 0.5 * dt * dt / (s44 * s44);
            M4 d_cov4{};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) d_cov4.a[a][b] = d_cov3_sym.a[a][b];
            for (int a = 0; a < 3; ++a) d_cov4.a[a][3] = d_cross[a];
            d_cov4.a[3][3] = d_s44;
            const double* ls = &v.s->log_s4[i * 4];
            double es4[4] = {std::exp(ls[0]), std::exp(ls[1]), std::exp(ls[2]), std::exp(ls[3])};
            M4 m4;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) m4.a[a][b] = pt.rot4.a[a][b] * es4[b];
            M4 sym;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) sym.a[a][b] = d_cov4.a[a][b] + d_cov4.a[b][a];
            M4 d_m4 = mul4(sym, m4);
            for (int k = 0; k < 4; ++k) {
                double a = 0.0;
                for (int r = 0; r < 4; ++r) a += d_m4.a[r][k] * m4.a[r][k];
                G.log_s4[i * 4 + k] += a;
            }
            M4 d_rot4;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) d_rot4.a[a][b] = d_m4.a[a][b] * es4[b];
            const double* ql = &v.s->ql[i * 4];
            const double* qr = &v.s->qr[i * 4];
            M4 rmat = right_isoclinic(qr), lmat = left_isoclinic(ql);
            M4 d_lmat, d_rmat;
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) {
                    double x = 0.0, y = 0.0;
                    for (int k = 0; k < 4; ++k) {
                        x += d_rot4.a[a][k] * rmat.a[b][k];  // d_rot4 * rmat^T
                        y += lmat.a[k][a] * d_rot4.a[k][b];  // lmat^T * d_rot4
                    }
                    d_lmat.a[a][b] = x;
                    d_rmat.a[a][b] = y;
                }
            double dql[4], dqr[4];
            for (int k = 0; k < 4; ++k) {
                double ek[4] = {double(k == 0), double(k == 1), double(k == 2), double(k == 3)};
                M4 le = left_isoclinic(ek), re = right_isoclinic(ek);
                double x = 0.0, y = 0.0;
                for (int a = 0; a < 4; ++a)
                    for (int b = 0; b < 4; ++b) {
                        x += d_lmat.a[a][b] * le.a[a][b];
                        y += d_rmat.a[a][b] * re.a[a][b];
                    }
                dql[k] = x;
                dqr[k] = y;
            }
            double tl[4], trr[4];
            through_normalization(ql, dql, tl);
            through_normalization(qr, dqr, trr);
            for (int k = 0; k < 4; ++k) {
                G.ql[i * 4 + k] += tl[k];
                G.qr[i * 4 + k] += trr[k];
            }
        }
    }
}

// backward.cpp:17-40
void grads_add_scaled(const hgso_scene& shape, hgso_grads& a, const hgso_grads& b, double scale) {
    const int K3 = sh_count(shape.sh_degree) * 3;
    const int64_t n3 = shape.n3, n4 = shape.n4;
    for (int64_t i = 0; i < n3; ++i) {
        for (int k = 0; k < 3; ++k) a.mean3[i * 3 + k] += scale * b.mean3[i * 3 + k];
        for (int k = 0; k < 4; ++k) a.quat3[i * 4 + k] += scale * b.quat3[i * 4 + k];
        for (int k = 0; k < 3; ++k) a.log_s3[i * 3 + k] += scale * b.log_s3[i * 3 + k];
        a.op3[i] += scale * b.op3[i];
        for (int k = 0; k < K3; ++k) a.sh3[i * K3 + k] += scale * b.sh3[i * K3 + k];
        a.screen_norm3[i] += b.screen_norm3[i];
    }
    for (int64_t i = 0; i < n4; ++i) {
        for (int k = 0; k < 3; ++k) a.mean_x[i * 3 + k] += scale * b.mean_x[i * 3 + k];
        a.mean_t[i] += scale * b.mean_t[i];
        for (int k = 0; k < 4; ++k) a.ql[i * 4 + k] += scale * b.ql[i * 4 + k];
        for (int k = 0; k < 4; ++k) a.qr[i * 4 + k] += scale * b.qr[i * 4 + k];
        for (int k = 0; k < 4; ++k) a.log_s4[i * 4 + k] += scale * b.log_s4[i * 4 + k];
        a.op4[i] += scale * b.op4[i];
        for (int k = 0; k < K3; ++k) a.sh4[i * K3 + k] += scale * b.sh4[i * K3 + k];
        a.screen_norm4[i] += b.screen_norm4[i];
    }
}

// ------------------------------------------------------------ loss / metrics
constexpr int kWin = 11;
constexpr double kSigma = 1.5;
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;

// metrics.cpp:16-30
const std::vector<double>& ssim_window() {
    static const std::vector<double> w = [] {
        std::vector<double> out(kWin * kWin);
        double sum = 0.0;
        for (int i = 0; i < kWin; ++i)
            for (int j = 0; j < kWin; ++j) {
                double di = i - kWin / 2, dj = j - kWin / 2;
                out[i * kWin + j] = std::exp(-(di * di + dj * dj) / (2.0 * kSigma * kSigma));
                sum += out[i * kWin + j];
            }
        for (double& v : out) v /= sum;
        return out;
    }();
    return w;
}

// metrics.cpp:37-87
double ssim_impl(const double* a, const double* b, int W, int H, double* grad) {
    if (W < kWin || H < kWin) throw std::invalid_argument("ssim: images smaller than the 11x11 window");
    const auto& w = ssim_window();
    const int vw = W - kWin + 1, vh = H - kWin + 1;
    const double n_valid = double(size_t(vw) * vh * 3);
    auto at = [&](const double* img, int x, int y, int c) { return img[(size_t(y) * W + x) * 3 + c]; };
    double total = 0.0;
    for (int c = 0; c < 3; ++c)
        for (int vy = 0; vy < vh; ++vy)
            for (int vx = 0; vx < vw; ++vx) {
                double mu_a = 0, mu_b = 0, aa = 0, bb = 0, ab = 0;
                for (int i = 0; i < kWin; ++i)
                    for (int j = 0; j < kWin; ++j) {
                        double wi = w[i * kWin + j];
                        double va = at(a, vx + j, vy + i, c), vb = at(b, vx + j, vy + i, c);
                        mu_a += wi * va;
                        mu_b += wi * vb;
                        aa += wi * va * va;
                        bb += wi * vb * vb;
                        ab += wi * va * vb;
                    }
                double var_a = aa - mu_a * mu_a, var_b = bb - mu_b * mu_b, cov = ab - mu_a * mu_b;
                double a1 = 2.0 * mu_a * mu_b + kC1, a2 = 2.0 * cov + kC2;
                double b1 = mu_a * mu_a + mu_b * mu_b + kC1, b2 = var_a + var_b + kC2;
                double denom = b1 * b2;
                double s = a1 * a2 / denom;
                total += s;
                if (grad) {
                    double d_mu = (a2 / denom) * 2.0 * mu_b - (s / b1) * 2.0 * mu_a;
                    double d_var = -s / b2;
                    double d_cov = 2.0 * a1 / denom;
                    for (int i = 0; i < kWin; ++i)
                        for (int j = 0; j < kWin; ++j) {
                            double wi = w[i * kWin + j];
                            double va = at(a, vx + j, vy + i, c), vb = at(b, vx + j, vy + i, c);
                            grad[(size_t(vy + i) * W + vx + j) * 3 + c] +=
                                wi * (d_mu + d_var * 2.0 * (va - mu_a) + d_cov * (vb - mu_b)) / n_valid;
                        }
                }
            }
    return total / n_valid;
}

// loss.cpp:13-22
double l1(const double* a, const double* b, size_t n, double* grad) {
    double sum = 0.0;
    const double dn = double(n);
    for (size_t i = 0; i < n; ++i) {
        double d = a[i] - b[i];
        sum += std::abs(d);
        if (grad) grad[i] = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / dn;
    }
    return sum / dn;
}

// metrics.cpp:91-101
double psnr(const double* a, const double* b, size_t n) {
    double mse = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double d = a[i] - b[i];
        mse += d * d;
    }
    mse /= double(n);
    if (mse == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(1.0 / mse);
}

// ------------------------------------------------------------ optimizer
constexpr double kBeta1 = 0.9, kBeta2 = 0.999, kEps = 1e-15;  // train.cpp:18-20

bool all_finite(const double* g, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(g[i])) return false;
    return true;
}
// train.cpp:29-42
void adam_row(double* value, const double* grad, double* m, double* v, size_t dim, double lr,
              double bc1, double bc2, uint64_t* skipped) {
    if (!all_finite(grad, dim)) {
        (*skipped)++;
        return;
    }
    for (size_t k = 0; k < dim; ++k) {
        m[k] = kBeta1 * m[k] + (1.0 - kBeta1) * grad[k];
        v[k] = kBeta2 * v[k] + (1.0 - kBeta2) * grad[k] * grad[k];
        double mhat = m[k] / bc1;
        double vhat = v[k] / bc2;
        value[k] -= lr * mhat / (std::sqrt(vhat) + kEps);
    }
}
// train.cpp:46-53
void renorm_quat(double* raw, double* m) {
    double n = std::sqrt(raw[0] * raw[0] + raw[1] * raw[1] + raw[2] * raw[2] + raw[3] * raw[3]);
    double w = raw[0] / n, x = raw[1] / n, y = raw[2] / n, z = raw[3] / n;
    bool flip = w < 0.0 || (w == 0.0 && (x < 0.0 || (x == 0.0 && (y < 0.0 || (y == 0.0 && z < 0.0)))));
    if (flip)
        for (int k = 0; k < 4; ++k) m[k] = -m[k];
    quat_normalized(w, x, y, z, raw);
}

// train.cpp:131-180
void optimizer_step(hgso_scene& s, const hgso_grads& g, hgso_state& st, const hgso_lrs& lrs,
                    double mean_lr_scale) {
    st.step++;
    const double bc1 = 1.0 - std::pow(kBeta1, double(st.step));
    const double bc2 = 1.0 - std::pow(kBeta2, double(st.step));
    const size_t sh_dim = 3 * size_t(sh_count(s.sh_degree));
    const double lr_mean = lrs.mean * s.extent * mean_lr_scale;
    const double lr_mean_t = lrs.mean_t * mean_lr_scale;
    uint64_t* sk = &st.skipped_nonfinite;
    hgso_scene& M = st.m;
    hgso_scene& V = st.v;
    for (int64_t i = 0; i < s.n3; ++i) {
        adam_row(&s.mean3[i * 3], &g.mean3[i * 3], &M.mean3[i * 3], &V.mean3[i * 3], 3, lr_mean, bc1, bc2, sk);
        adam_row(&s.quat3[i * 4], &g.quat3[i * 4], &M.quat3[i * 4], &V.quat3[i * 4], 4, lrs.quat, bc1, bc2, sk);
        renorm_quat(&s.quat3[i * 4], &M.quat3[i * 4]);
        adam_row(&s.log_s3[i * 3], &g.log_s3[i * 3], &M.log_s3[i * 3], &V.log_s3[i * 3], 3, lrs.scales, bc1, bc2, sk);
        adam_row(&s.op3[i], &g.op3[i], &M.op3[i], &V.op3[i], 1, lrs.opacity, bc1, bc2, sk);
        adam_row(&s.sh3[i * sh_dim], &g.sh3[i * sh_dim], &M.sh3[i * sh_dim], &V.sh3[i * sh_dim], sh_dim, lrs.sh, bc1, bc2, sk);
    }
    for (int64_t i = 0; i < s.n4; ++i) {
        adam_row(&s.mean_x[i * 3], &g.mean_x[i * 3], &M.mean_x[i * 3], &V.mean_x[i * 3], 3, lr_mean, bc1, bc2, sk);
        adam_row(&s.mean_t[i], &g.mean_t[i], &M.mean_t[i], &V.mean_t[i], 1, lr_mean_t, bc1, bc2, sk);
        adam_row(&s.ql[i * 4], &g.ql[i * 4], &M.ql[i * 4], &V.ql[i * 4], 4, lrs.quat, bc1, bc2, sk);
        renorm_quat(&s.ql[i * 4], &M.ql[i * 4]);
        adam_row(&s.qr[i * 4], &g.qr[i * 4], &M.qr[i * 4], &V.qr[i * 4], 4, lrs.quat, bc1, bc2, sk);
        renorm_quat(&s.qr[i * 4], &M.qr[i * 4]);
        adam_row(&s.log_s4[i * 4], &g.log_s4[i * 4], &M.log_s4[i * 4], &V.log_s4[i * 4], 4, lrs.scales, bc1, bc2, sk);
        adam_row(&s.op4[i], &g.op4[i], &M.op4[i], &V.op4[i], 1, lrs.opacity, bc1, bc2, sk);
        adam_row(&s.sh4[i * sh_dim], &g.sh4[i * sh_dim], &M.sh4[i * sh_dim], &V.sh4[i * sh_dim], sh_dim, lrs.sh, bc1, bc2, sk);
    }
}

// ------------------------------------------------------------ conversion
// scene.cpp:19-31
double mean_temporal_weight(double mean_t, double sigma_t) {
    const double s = sigma_t * std::sqrt(2.0);
    double w = sigma_t * std::sqrt(M_PI / 2.0) * (std::erf((1.0 - mean_t) / s) + std::erf(mean_t / s));
    return w < 1.0 ? w : 1.0;
}
double fold_temporal_weight(double opacity_logit, double mean_t, double sigma_t) {
    double w = mean_temporal_weight(mean_t, sigma_t);
    if (w >= 1.0 - 1e-12) return opacity_logit;
    double alpha = sigmoid(opacity_logit) * w;
    return std::log(alpha) - std::log1p(-alpha);
}

// scene.cpp:10-13
bool is_static(double log_st, double tau) {
    if (!(tau > 0.0)) throw std::invalid_argument("is_static: tau must be positive");
    return std::exp(log_st) > tau;
}

// scene.cpp:33-41 (also the body of sweep_convert's loop, 50-58)
double convert_one(const hgso_scene& s, int64_t i, double mean3[3], double quat[4], double ls3[3],
                   double* op) {
    M4 r4 = rot4_from_pair(&s.ql[i * 4], &s.qr[i * 4]);
    M3 rot;
    double leakage;
    extract_spatial_rot(r4, rot, leakage);
    for (int k = 0; k < 3; ++k) mean3[k] = s.mean_x[i * 3 + k];
    rot3_to_quat(rot, quat);
    for (int k = 0; k < 3; ++k) ls3[k] = s.log_s4[i * 4 + k];
    *op = fold_temporal_weight(s.op4[i], s.mean_t[i], std::exp(s.log_s4[i * 4 + 3]));
    return leakage;
}

// scene.cpp:43-71 + train.cpp:305-362 (remap_after_sweep), in place.
void sweep_convert(hgso_scene& s, hgso_state* st, int64_t* moved, hgso_conversion& rep) {
    const int K3 = sh_count(s.sh_degree) * 3;
    rep.count = 0;
    rep.max_leakage = 0.0;
    rep.mean_leakage = 0.0;
    double leak_sum = 0.0;
    const int64_t n4 = s.n4, n3_before = s.n3;
    std::vector<int64_t> mv;
    std::vector<char> is_moved(size_t(n4), 0);
    for (int64_t i = 0; i < n4; ++i) {
        if (!is_static(s.log_s4[i * 4 + 3], s.tau)) continue;
        int64_t dst = n3_before + int64_t(mv.size());
        double leak = convert_one(s, i, &s.mean3[dst * 3], &s.quat3[dst * 4], &s.log_s3[dst * 3], &s.op3[dst]);
        for (int k = 0; k < K3; ++k) s.sh3[dst * K3 + k] = s.sh4[i * K3 + k];
        rep.count++;
        rep.max_leakage = std::max(rep.max_leakage, leak);
        leak_sum += leak;
        mv.push_back(i);
        is_moved[size_t(i)] = 1;
    }
    if (rep.count > 0) rep.mean_leakage = leak_sum / double(rep.count);
    if (st) {  // train.cpp:323-341 moment inheritance: mean_x, scales[0:3], quat_left, opacity, SH
        for (size_t k = 0; k < mv.size(); ++k) {
            int64_t dst = n3_before + int64_t(k), src = mv[k];
            for (hgso_scene* B : {&st->m, &st->v}) {
                for (int c = 0; c < 3; ++c) B->mean3[dst * 3 + c] = B->mean_x[src * 3 + c];
                for (int c = 0; c < 3; ++c) B->log_s3[dst * 3 + c] = B->log_s4[src * 4 + c];
                for (int c = 0; c < 4; ++c) B->quat3[dst * 4 + c] = B->ql[src * 4 + c];
                B->op3[dst] = B->op4[src];
                for (int c = 0; c < K3; ++c) B->sh3[dst * K3 + c] = B->sh4[src * K3 + c];
            }
        }
    }
    // stable compaction of the survivors (scene.cpp:59-61; train.cpp:343-355)
    auto compact = [&](hgso_scene& P) {
        int64_t w = 0;
        for (int64_t i = 0; i < n4; ++i) {
            if (is_moved[size_t(i)]) continue;
            if (w != i) {
                for (int c = 0; c < 3; ++c) P.mean_x[w * 3 + c] = P.mean_x[i * 3 + c];
                P.mean_t[w] = P.mean_t[i];
                for (int c = 0; c < 4; ++c) P.ql[w * 4 + c] = P.ql[i * 4 + c];
                for (int c = 0; c < 4; ++c) P.qr[w * 4 + c] = P.qr[i * 4 + c];
                for (int c = 0; c < 4; ++c) P.log_s4[w * 4 + c] = P.log_s4[i * 4 + c];
                P.op4[w] = P.op4[i];
                for (int c = 0; c < K3; ++c) P.sh4[w * K3 + c] = P.sh4[i * K3 + c];
            }
            ++w;
        }
    };
    compact(s);
    if (st) {
        compact(st->m);
        compact(st->v);
    }
    s.n4 = n4 - int64_t(mv.size());
    s.n3 = n3_before + int64_t(mv.size());
    if (st) {  // train.cpp:357-361: every densify statistic is reset
        for (int64_t i = 0; i < s.n3; ++i) { st->grad_norm3[i] = 0.0; st->count3[i] = 0; }
        for (int64_t i = 0; i < s.n4; ++i) { st->grad_norm4[i] = 0.0; st->count4[i] = 0; }
    }
    for (size_t k = 0; k < mv.size(); ++k) moved[k] = mv[k];
}

// ------------------------------------------------------------ C boundary helpers
template <typename F>
int guard(F&& f) {
    try {
        f();
        return HGSO_OK;
    } catch (const DegenerateTemporal& e) {
        g_err = e.what();
        return HGSO_DEGENERATE_TEMPORAL;
    } catch (const DegenerateRotation& e) {
        g_err = e.what();
        return HGSO_DEGENERATE_ROTATION;
    } catch (const NumericAbort& e) {
        g_err = e.what();
        return HGSO_NUMERIC_ABORT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HGSO_INVALID_ARGUMENT;
    }
}

}  // namespace hgso

using namespace hgso;

extern "C" {

const char* hgso_last_error(void) { return g_err.c_str(); }

void* hgso_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void hgso_rng_free(void* rng) { delete static_cast<std::mt19937_64*>(rng); }
double hgso_rng_uniform(void* rng) {
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    return uni(*static_cast<std::mt19937_64*>(rng));
}
double hgso_rng_normal(void* rng) {
    std::normal_distribution<double> nd(0.0, 1.0);
    return nd(*static_cast<std::mt19937_64*>(rng));
}
// train.cpp:392 `std::uniform_int_distribution<std::size_t> pick(0, n - 1)`
uint64_t hgso_rng_index(void* rng, uint64_t lo, uint64_t hi) {
    std::uniform_int_distribution<std::size_t> pick(lo, hi);
    return pick(*static_cast<std::mt19937_64*>(rng));
}
uint64_t hgso_rng_raw(void* rng) { return (*static_cast<std::mt19937_64*>(rng))(); }
void hgso_rng_normal_seq(void* rng, int64_t n, double* out) {
    std::normal_distribution<double> nd(0.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = nd(*static_cast<std::mt19937_64*>(rng));
}

// train.cpp:182-299 densify_and_prune, restated on the flat pools.  Per pool,
// in index order: prune if sigmoid(opacity) < eps; "dense" if the averaged
// screen gradient exceeds the threshold and two more rows still fit under
// max_gaussians; dense and small (max scale < clone_size_frac * extent) ->
// the original + a clone jittered by 0.1 * (R diag(e^s)) n; dense and large
// -> two parts offset by (R diag(e^s)) n with scales / split_factor.  Normal
// draws: statics call sample_normal3 (a fresh normal_distribution per call,
// train.cpp:68-72); dynamics share one distribution for the whole pool and
// fill Vec4(nd, nd, nd, nd), whose arguments g++ evaluates right to left.
// Adam rows follow their source (remap_buf, train.cpp:56-66: fresh rows 0).
int hgso_densify_and_prune(const hgso_scene* in, const hgso_state* st_in, hgso_scene* out, hgso_state* st_out,
                           const hgso_densify_cfg* cfg, void* rngp, hgso_densify_report* rep) {
    return guard([&] {
        auto& rng = *static_cast<std::mt19937_64*>(rngp);
        *rep = hgso_densify_report{};
        const int K3 = 3 * sh_count(in->sh_degree);
        const double size_gate = cfg->clone_size_frac * in->extent;
        const double log_split = std::log(cfg->split_factor);
        const size_t maxg = size_t(cfg->max_gaussians);
        auto sig = [](double x) { return 1.0 / (1.0 + std::exp(-x)); };
        // ---- statics
        {
            size_t o = 0;
            auto copy_row = [&](int64_t i, size_t d, bool adam) {
                for (int k = 0; k < 3; ++k) out->mean3[d * 3 + k] = in->mean3[i * 3 + k];
                for (int k = 0; k < 4; ++k) out->quat3[d * 4 + k] = in->quat3[i * 4 + k];
                for (int k = 0; k < 3; ++k) out->log_s3[d * 3 + k] = in->log_s3[i * 3 + k];
                out->op3[d] = in->op3[i];
                for (int k = 0; k < K3; ++k) out->sh3[d * K3 + k] = in->sh3[i * K3 + k];
                const hgso_scene* sm[2] = {&st_in->m, &st_in->v};
                hgso_scene* dm[2] = {&st_out->m, &st_out->v};
                for (int b = 0; b < 2; ++b) {
                    for (int k = 0; k < 3; ++k) dm[b]->mean3[d * 3 + k] = adam ? sm[b]->mean3[i * 3 + k] : 0.0;
                    for (int k = 0; k < 4; ++k) dm[b]->quat3[d * 4 + k] = adam ? sm[b]->quat3[i * 4 + k] : 0.0;
                    for (int k = 0; k < 3; ++k) dm[b]->log_s3[d * 3 + k] = adam ? sm[b]->log_s3[i * 3 + k] : 0.0;
                    dm[b]->op3[d] = adam ? sm[b]->op3[i] : 0.0;
                    for (int k = 0; k < K3; ++k) dm[b]->sh3[d * K3 + k] = adam ? sm[b]->sh3[i * K3 + k] : 0.0;
                }
            };
            auto sample_normal3 = [&](double n[3]) {
                std::normal_distribution<double> nd(0.0, 1.0);
                double a = nd(rng), b = nd(rng), c = nd(rng);
                n[0] = a;
                n[1] = b;
                n[2] = c;
            };
            for (int64_t i = 0; i < in->n3; ++i) {
                if (sig(in->op3[i]) < cfg->opacity_prune_eps) {
                    rep->pruned3++;
                    continue;
                }
                const double avg = st_in->count3[i] > 0 ? st_in->grad_norm3[i] / st_in->count3[i] : 0.0;
                const bool dense = avg > cfg->grad_threshold && o + 2 <= maxg;
                const double* ls = &in->log_s3[i * 3];
                const double mx = std::max(std::max(std::exp(ls[0]), std::exp(ls[1])), std::exp(ls[2]));
                if (dense) {
                    const M3 r = quat_to_rot3(&in->quat3[i * 4]);
                    double m[3][3];
                    for (int a = 0; a < 3; ++a)
                        for (int b = 0; b < 3; ++b) m[a][b] = r.a[a][b] * std::exp(ls[b]);
                    auto mv = [&](const double n[3], double y[3]) {
                        for (int a = 0; a < 3; ++a) y[a] = m[a][0] * n[0] + m[a][1] * n[1] + m[a][2] * n[2];
                    };
                    if (mx < size_gate) {
                        copy_row(i, o, true);
                        double n[3], y[3];
                        sample_normal3(n);
                        mv(n, y);
                        copy_row(i, o + 1, false);
                        for (int a = 0; a < 3; ++a) out->mean3[(o + 1) * 3 + a] = in->mean3[i * 3 + a] + 0.1 * y[a];
                        o += 2;
                        rep->cloned3++;
                    } else {
                        for (int c = 0; c < 2; ++c) {
                            double n[3], y[3];
                            sample_normal3(n);
                            mv(n, y);
                            copy_row(i, o, false);
                            for (int a = 0; a < 3; ++a) out->mean3[o * 3 + a] = in->mean3[i * 3 + a] + y[a];
                            for (int a = 0; a < 3; ++a) out->log_s3[o * 3 + a] = ls[a] - log_split;
                            ++o;
                        }
                        rep->split3++;
                    }
                } else {
                    copy_row(i, o, true);
                    ++o;
                }
            }
            out->n3 = int64_t(o);
            for (size_t k = 0; k < o; ++k) {
                st_out->grad_norm3[k] = 0.0;
                st_out->count3[k] = 0;
            }
        }
        // ---- dynamics
        {
            size_t o = 0;
            std::normal_distribution<double> nd(0.0, 1.0);
            auto copy_row = [&](int64_t i, size_t d, bool adam) {
                for (int k = 0; k < 3; ++k) out->mean_x[d * 3 + k] = in->mean_x[i * 3 + k];
                out->mean_t[d] = in->mean_t[i];
                for (int k = 0; k < 4; ++k) out->ql[d * 4 + k] = in->ql[i * 4 + k];
                for (int k = 0; k < 4; ++k) out->qr[d * 4 + k] = in->qr[i * 4 + k];
                for (int k = 0; k < 4; ++k) out->log_s4[d * 4 + k] = in->log_s4[i * 4 + k];
                out->op4[d] = in->op4[i];
                for (int k = 0; k < K3; ++k) out->sh4[d * K3 + k] = in->sh4[i * K3 + k];
                const hgso_scene* sm[2] = {&st_in->m, &st_in->v};
                hgso_scene* dm[2] = {&st_out->m, &st_out->v};
                for (int b = 0; b < 2; ++b) {
                    for (int k = 0; k < 3; ++k) dm[b]->mean_x[d * 3 + k] = adam ? sm[b]->mean_x[i * 3 + k] : 0.0;
                    dm[b]->mean_t[d] = adam ? sm[b]->mean_t[i] : 0.0;
                    for (int k = 0; k < 4; ++k) dm[b]->ql[d * 4 + k] = adam ? sm[b]->ql[i * 4 + k] : 0.0;
                    for (int k = 0; k < 4; ++k) dm[b]->qr[d * 4 + k] = adam ? sm[b]->qr[i * 4 + k] : 0.0;
                    for (int k = 0; k < 4; ++k) dm[b]->log_s4[d * 4 + k] = adam ? sm[b]->log_s4[i * 4 + k] : 0.0;
                    dm[b]->op4[d] = adam ? sm[b]->op4[i] : 0.0;
                    for (int k = 0; k < K3; ++k) dm[b]->sh4[d * K3 + k] = adam ? sm[b]->sh4[i * K3 + k] : 0.0;
                }
            };
            auto draw4 = [&](double n[4]) {  // Vec4 n(nd(rng), nd(rng), nd(rng), nd(rng)), g++ right-to-left
                const double d0 = nd(rng), d1 = nd(rng), d2 = nd(rng), d3 = nd(rng);
                n[0] = d3;
                n[1] = d2;
                n[2] = d1;
                n[3] = d0;
            };
            for (int64_t i = 0; i < in->n4; ++i) {
                if (sig(in->op4[i]) < cfg->opacity_prune_eps) {
                    rep->pruned4++;
                    continue;
                }
                const double avg = st_in->count4[i] > 0 ? st_in->grad_norm4[i] / st_in->count4[i] : 0.0;
                const bool dense = avg > cfg->grad_threshold && o + 2 <= maxg;
                const double* ls = &in->log_s4[i * 4];
                const double mx = std::max(std::max(std::exp(ls[0]), std::exp(ls[1])), std::exp(ls[2]));
                if (dense) {
                    const M4 r = rot4_from_pair(&in->ql[i * 4], &in->qr[i * 4]);
                    double m[4][4];
                    for (int a = 0; a < 4; ++a)
                        for (int b = 0; b < 4; ++b) m[a][b] = r.a[a][b] * std::exp(ls[b]);
                    auto mv = [&](const double n[4], double y[4]) {
                        for (int a = 0; a < 4; ++a)
                            y[a] = m[a][0] * n[0] + m[a][1] * n[1] + m[a][2] * n[2] + m[a][3] * n[3];
                    };
                    if (mx < size_gate) {
                        copy_row(i, o, true);
                        double n[4], y[4];
                        draw4(n);
                        mv(n, y);
                        copy_row(i, o + 1, false);
                        for (int a = 0; a < 3; ++a) out->mean_x[(o + 1) * 3 + a] = in->mean_x[i * 3 + a] + 0.1 * y[a];
                        o += 2;
                        rep->cloned4++;
                    } else {
                        for (int c = 0; c < 2; ++c) {
                            double n[4], y[4];
                            draw4(n);
                            mv(n, y);
                            copy_row(i, o, false);
                            for (int a = 0; a < 3; ++a) out->mean_x[o * 3 + a] = in->mean_x[i * 3 + a] + y[a];
                            out->mean_t[o] = in->mean_t[i] + y[3];
                            for (int a = 0; a < 4; ++a) out->log_s4[o * 4 + a] = ls[a] - log_split;
                            ++o;
                        }
                        rep->split4++;
                    }
                } else {
                    copy_row(i, o, true);
                    ++o;
                }
            }
            out->n4 = int64_t(o);
            for (size_t k = 0; k < o; ++k) {
                st_out->grad_norm4[k] = 0.0;
                st_out->count4[k] = 0;
            }
        }
        out->sh_degree = in->sh_degree;
        out->tau = in->tau;
        out->extent = in->extent;
    });
}

// tests/oracles.hpp:26-29
void hgso_random_quat(void* rngp, double q[4]) {
    auto& rng = *static_cast<std::mt19937_64*>(rngp);
    std::normal_distribution<double> nd(0.0, 1.0);
    double d = nd(rng), c = nd(rng), b = nd(rng), a = nd(rng);  // g++: args right-to-left
    quat_normalized(a, b, c, d, q);
}

// tests/oracles.hpp:63-97.  The reference draws inside constructor argument
// lists, e.g. Vec3(nd(rng), nd(rng), nd(rng)); C++ leaves that order
// unspecified and g++ (the toolchain the reference targets) evaluates such
// arguments right to left, which is what is reproduced here draw for draw.
void hgso_random_scene(void* rngp, int n_static, int n_dynamic, int sh_degree, hgso_scene* out) {
    auto& rng = *static_cast<std::mt19937_64*>(rngp);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    const int K = sh_count(sh_degree);
    out->sh_degree = sh_degree;
    out->extent = 2.0;
    out->n3 = n_static;
    out->n4 = n_dynamic;
    auto sh_fill = [&](double* sh) {
        double b = uni(rng), g = uni(rng), r = uni(rng);
        for (int k = 0; k < K * 3; ++k) sh[k] = 0.0;
        sh[0] = (r - 0.5) / C0;
        sh[1] = (g - 0.5) / C0;
        sh[2] = (b - 0.5) / C0;
        for (int k = 1; k < K; ++k) {
            double z = nd(rng), y = nd(rng), x = nd(rng);
            sh[k * 3] = 0.2 * x;
            sh[k * 3 + 1] = 0.2 * y;
            sh[k * 3 + 2] = 0.2 * z;
        }
    };
    for (int i = 0; i < n_static; ++i) {
        double z = nd(rng), y = nd(rng), x = nd(rng);
        out->mean3[i * 3] = x * 1.2;
        out->mean3[i * 3 + 1] = y * 1.2;
        out->mean3[i * 3 + 2] = z * 1.2;
        hgso_random_quat(rngp, &out->quat3[i * 4]);
        double u2 = uni(rng), u1 = uni(rng), u0 = uni(rng);
        out->log_s3[i * 3] = std::log(0.05 + 0.3 * u0);
        out->log_s3[i * 3 + 1] = std::log(0.05 + 0.3 * u1);
        out->log_s3[i * 3 + 2] = std::log(0.05 + 0.3 * u2);
        out->op3[i] = logit(0.05 + 0.9 * uni(rng));
        sh_fill(&out->sh3[i * K * 3]);
    }
    for (int i = 0; i < n_dynamic; ++i) {
        double z = nd(rng), y = nd(rng), x = nd(rng);
        out->mean_x[i * 3] = x * 1.2;
        out->mean_x[i * 3 + 1] = y * 1.2;
        out->mean_x[i * 3 + 2] = z * 1.2;
        out->mean_t[i] = uni(rng);
        hgso_random_quat(rngp, &out->ql[i * 4]);
        hgso_random_quat(rngp, &out->qr[i * 4]);
        double u3 = uni(rng), u2 = uni(rng), u1 = uni(rng), u0 = uni(rng);
        out->log_s4[i * 4] = std::log(0.05 + 0.3 * u0);
        out->log_s4[i * 4 + 1] = std::log(0.05 + 0.3 * u1);
        out->log_s4[i * 4 + 2] = std::log(0.05 + 0.3 * u2);
        out->log_s4[i * 4 + 3] = std::log(0.08 + 0.5 * u3);
        out->op4[i] = logit(0.05 + 0.9 * uni(rng));
        sh_fill(&out->sh4[i * K * 3]);
    }
}

// tests/oracles.hpp:99-108
int hgso_random_camera(void* rngp, int width, int height, hgso_camera* out) {
    auto& rng = *static_cast<std::mt19937_64*>(rngp);
    return guard([&] {
        std::uniform_real_distribution<double> uni(0.0, 1.0);
        double a = 2.0 * M_PI * uni(rng);
        double h = -1.5 + 3.0 * uni(rng);
        double r = 4.0 + 2.0 * uni(rng);
        double eye[3] = {r * std::cos(a), h, r * std::sin(a)};
        double tgt[3] = {0, 0, 0}, up[3] = {0, -1, 0};
        Cam cam = look_at(eye, tgt, up, 60.0, width, height);
        validate(cam);
        *out = from_cam(cam);
    });
}

int hgso_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                 int width, int height, hgso_camera* out) {
    return guard([&] { *out = from_cam(look_at(eye, target, up, focal, width, height)); });
}

int hgso_quat_to_rot3(const double q[4], double r[9]) {
    return guard([&] {
        M3 m = quat_to_rot3(q);
        for (int i = 0; i < 9; ++i) r[i] = m.a[i / 3][i % 3];
    });
}
int hgso_rot3_to_quat(const double r[9], double q[4]) {
    return guard([&] {
        M3 m;
        for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = r[i];
        rot3_to_quat(m, q);
    });
}
void hgso_rot4_from_pair(const double ql[4], const double qr[4], double r[16]) {
    M4 m = rot4_from_pair(ql, qr);
    for (int i = 0; i < 16; ++i) r[i] = m.a[i / 4][i % 4];
}
void hgso_build_cov4(const double r[16], const double ls[4], double cov[16]) {
    M4 m;
    for (int i = 0; i < 16; ++i) m.a[i / 4][i % 4] = r[i];
    M4 c = build_cov4(m, ls);
    for (int i = 0; i < 16; ++i) cov[i] = c.a[i / 4][i % 4];
}
void hgso_build_cov3(const double r[9], const double ls[3], double cov[9]) {
    M3 m;
    for (int i = 0; i < 9; ++i) m.a[i / 3][i % 3] = r[i];
    M3 c = build_cov3(m, ls);
    for (int i = 0; i < 9; ++i) cov[i] = c.a[i / 3][i % 3];
}
int hgso_condition_at_time(const double mean4[4], const double cov4[16], double t, double mean3[3],
                           double cov3[9], double* weight) {
    return guard([&] {
        M4 c;
        for (int i = 0; i < 16; ++i) c.a[i / 4][i % 4] = cov4[i];
        Slice s = condition_at_time(mean4, c, t);
        for (int i = 0; i < 3; ++i) mean3[i] = s.mean3[i];
        for (int i = 0; i < 9; ++i) cov3[i] = s.cov3.a[i / 3][i % 3];
        *weight = s.weight;
    });
}
int hgso_clamp_psd(const double m[9], double eps, double out[9]) {
    return guard([&] {
        M3 a;
        for (int i = 0; i < 9; ++i) a.a[i / 3][i % 3] = m[i];
        M3 r = clamp_psd(a, eps);
        for (int i = 0; i < 9; ++i) out[i] = r.a[i / 3][i % 3];
    });
}
int hgso_extract_spatial_rot(const double r4[16], double r3[9], double* leakage) {
    return guard([&] {
        M4 m;
        for (int i = 0; i < 16; ++i) m.a[i / 4][i % 4] = r4[i];
        M3 r;
        extract_spatial_rot(m, r, *leakage);
        for (int i = 0; i < 9; ++i) r3[i] = r.a[i / 3][i % 3];
    });
}
void hgso_sh_basis(const double dir[3], int degree, double out[16]) {
    for (int i = 0; i < 16; ++i) out[i] = 0.0;
    sh_basis(dir, degree, out);
}
void hgso_sh_basis_grad(const double dir[3], int degree, double out[48]) { sh_basis_grad(dir, degree, out); }
int hgso_eval_sh(const double* coeffs, int degree, const double dir[3], double rgb[3]) {
    return guard([&] { eval_sh(coeffs, degree, dir, rgb); });
}
double hgso_exp(double x) { return std::exp(x); }

// raster.cpp:268-287 density_map: per pixel, the number of projected splats
// whose clamped box covers it (dynamics only on request).
int hgso_density_map(const hgso_scene* s, const hgso_camera* cam, double t, int dynamics_only, double cutoff,
                     uint32_t* counts) {
    return guard([&] {
        Cam c = to_cam(*cam);
        hgso_scene tmp = *s;
        if (dynamics_only) tmp.n3 = 0;
        View v{&tmp, sh_count(s->sh_degree)};
        std::vector<Splat> prims = project_scene(v, c, t, cutoff, nullptr);
        std::fill(counts, counts + size_t(c.width) * c.height, 0u);
        for (const Splat& sp : prims) {
            Bounds b = splat_bounds(sp, c.width, c.height);
            for (int y = b.y0; y <= b.y1; ++y)
                for (int x = b.x0; x <= b.x1; ++x) counts[size_t(y) * c.width + x]++;
        }
    });
}

// data_io.cpp:189-238 init_scene: one dynamic Gaussian per point; the
// literal serial O(N^2) 3-nearest-neighbour search.  out: n4 = n, n3 = 0,
// buffers sized by the caller.
int hgso_init_scene(const double* pos, const double* rgb, int64_t n, int sh_degree, double tau, double duration,
                    double init_temporal_scale, double init_opacity, hgso_scene* out, double* duration_out) {
    return guard([&] {
        if (n < 4) throw std::invalid_argument("init_scene: need at least 4 points");
        double c[3] = {0.0, 0.0, 0.0};
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) c[k] += pos[3 * i + k];
        for (int k = 0; k < 3; ++k) c[k] /= double(n);
        double extent = 1e-6;
        for (int64_t i = 0; i < n; ++i) {
            const double dx = pos[3 * i] - c[0], dy = pos[3 * i + 1] - c[1], dz = pos[3 * i + 2] - c[2];
            extent = std::max(extent, std::sqrt(dx * dx + dy * dy + dz * dz));
        }
        out->n4 = n;
        out->n3 = 0;
        out->sh_degree = sh_degree;
        out->tau = tau;
        out->extent = extent;
        *duration_out = duration;
        const int K = sh_count(sh_degree);
        const double nd = double(n);
        for (int64_t i = 0; i < n; ++i) {
            double d1 = 1e30, d2 = 1e30, d3 = 1e30;
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                const double dx = pos[3 * j] - pos[3 * i], dy = pos[3 * j + 1] - pos[3 * i + 1],
                             dz = pos[3 * j + 2] - pos[3 * i + 2];
                const double d = dx * dx + dy * dy + dz * dz;
                if (d < d1) { d3 = d2; d2 = d1; d1 = d; }
                else if (d < d2) { d3 = d2; d2 = d; }
                else if (d < d3) { d3 = d; }
            }
            const double mean_nn = (std::sqrt(d1) + std::sqrt(d2) + std::sqrt(d3)) / 3.0;
            const double s = std::log(std::max(mean_nn, 1e-4));
            for (int k = 0; k < 3; ++k) out->mean_x[3 * i + k] = pos[3 * i + k];
            out->mean_t[i] = (double(i) + 0.5) / nd;
            const double q[4] = {1.0, 0.0, 0.0, 0.0};
            for (int k = 0; k < 4; ++k) out->ql[4 * i + k] = out->qr[4 * i + k] = q[k];
            out->log_s4[4 * i + 0] = out->log_s4[4 * i + 1] = out->log_s4[4 * i + 2] = s;
            out->log_s4[4 * i + 3] = std::log(init_temporal_scale);
            out->op4[i] = std::log(init_opacity / (1.0 - init_opacity));
            double* sh = out->sh4 + size_t(i) * K * 3;
            std::fill(sh, sh + size_t(K) * 3, 0.0);
            for (int k = 0; k < 3; ++k) sh[k] = (rgb[3 * i + k] - 0.5) / C0;  // from_rgb_dc (sh.cpp:19-23)
        }
    });
}

static void fill_splat(const Splat& s, int n4, int W, int H, hgso_splat& o) {
    o.sx = s.sx; o.sy = s.sy;
    o.conic[0] = s.conic[0][0]; o.conic[1] = s.conic[0][1];
    o.conic[2] = s.conic[1][0]; o.conic[3] = s.conic[1][1];
    o.depth = s.depth;
    for (int c = 0; c < 3; ++c) o.rgb[c] = s.rgb[c];
    o.alpha = s.alpha;
    o.radius = s.radius;
    o.pool = s.pool;
    o.index = int32_t(s.index);
    o.gid = s.pool == 1 ? int32_t(s.index) : int32_t(n4 + int64_t(s.index));
    Bounds b = splat_bounds(s, W, H);
    o.x0 = b.x0; o.x1 = b.x1; o.y0 = b.y0; o.y1 = b.y1;
    o.depth_bits = f32_bits(s.depth);
    o.pad_ = 0;
}

int hgso_project_3d(const double mean3[3], const double cov3[9], const hgso_camera* cam,
                    hgso_splat* out, hgso_stats* stats, int* projected) {
    return guard([&] {
        Cam c = to_cam(*cam);
        M3 cv;
        for (int i = 0; i < 9; ++i) cv.a[i / 3][i % 3] = cov3[i];
        Splat s{};
        bool ok = project_3d(mean3, cv, c, stats, s);
        *projected = ok ? 1 : 0;
        if (ok) fill_splat(s, 0, c.width, c.height, *out);
    });
}

int hgso_project_scene(const hgso_scene* s, const hgso_camera* cam, double t, double cutoff,
                       hgso_splat* out, int64_t cap, int64_t* n_out, hgso_stats* stats) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        Cam c = to_cam(*cam);
        hgso_stats st{};
        std::vector<Splat> prims = project_scene(v, c, t, cutoff, &st);
        if (int64_t(prims.size()) > cap) throw std::invalid_argument("project_scene: output too small");
        for (size_t i = 0; i < prims.size(); ++i) fill_splat(prims[i], int(s->n4), c.width, c.height, out[i]);
        *n_out = int64_t(prims.size());
        if (stats) *stats = st;
    });
}

int hgso_sorted_instances(const hgso_scene* s, const hgso_camera* cam, double t, double cutoff,
                          uint32_t* tile_out, uint32_t* prim_out, int64_t cap, int64_t* n_out) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        Cam c = to_cam(*cam);
        std::vector<Splat> prims = project_scene(v, c, t, cutoff, nullptr);
        std::vector<Instance> inst;
        std::vector<std::pair<size_t, size_t>> ranges;
        int tiles_x;
        build_instances(prims, c, inst, ranges, tiles_x);
        *n_out = int64_t(inst.size());
        if (int64_t(inst.size()) > cap) return;
        for (size_t i = 0; i < inst.size(); ++i) {
            tile_out[i] = uint32_t(inst[i].key >> 32);
            prim_out[i] = inst[i].prim;
        }
    });
}

int hgso_rasterize(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3],
                   double cutoff, int num_threads, double* rgb, uint32_t* counts, double* trans,
                   hgso_stats* stats) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        Cam c = to_cam(*cam);
        size_t npx = size_t(c.width) * c.height;
        if (counts) std::fill(counts, counts + npx, 0u);
        if (trans) std::fill(trans, trans + npx, 1.0);
        rasterize(v, c, t, bg, cutoff, num_threads, rgb, counts, trans, stats);
    });
}

int hgso_reference_render(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3],
                          double cutoff, double* rgb, hgso_stats* stats) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        reference_render(v, to_cam(*cam), t, bg, cutoff, rgb, stats);
    });
}

int hgso_forward_train(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3],
                       double cutoff, int num_threads, double* rgb, void** tape_out) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        *tape_out = forward_train_tiled(v, to_cam(*cam), t, bg, cutoff, num_threads, rgb);
    });
}
int hgso_forward_train_untiled(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3],
                               double cutoff, double* rgb, void** tape_out) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        *tape_out = forward_train_untiled(v, to_cam(*cam), t, bg, cutoff, rgb);
    });
}
void hgso_tape_free(void* tape) { delete static_cast<Tape*>(tape); }
int64_t hgso_tape_contrib_total(void* tape) {
    int64_t n = 0;
    for (const auto& l : static_cast<Tape*>(tape)->contribs) n += int64_t(l.size());
    return n;
}
int hgso_backward(const hgso_scene* s, const hgso_camera* cam, void* tape, const double* loss_grad,
                  hgso_grads* g) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        backward(v, to_cam(*cam), *static_cast<Tape*>(tape), loss_grad, *g);
    });
}
void hgso_grads_add_scaled(const hgso_scene* shape, hgso_grads* acc, const hgso_grads* other, double scale) {
    grads_add_scaled(*shape, *acc, *other, scale);
}

// loss.cpp:26-49
double hgso_photometric_loss(const double* a, const double* b, int w, int h, double lambda) {
    size_t n = size_t(w) * h * 3;
    double loss = (1.0 - lambda) * l1(a, b, n, nullptr);
    if (lambda != 0.0) loss += lambda * (1.0 - ssim_impl(a, b, w, h, nullptr));
    return loss;
}
double hgso_photometric_loss_with_grad(const double* a, const double* b, int w, int h, double lambda,
                                       double* grad) {
    size_t n = size_t(w) * h * 3;
    double loss = (1.0 - lambda) * l1(a, b, n, grad);
    for (size_t i = 0; i < n; ++i) grad[i] *= (1.0 - lambda);
    if (lambda != 0.0) {
        std::vector<double> sg(n, 0.0);
        double s = ssim_impl(a, b, w, h, sg.data());
        loss += lambda * (1.0 - s);
        for (size_t i = 0; i < n; ++i) grad[i] -= lambda * sg[i];
    }
    return loss;
}
double hgso_ssim(const double* a, const double* b, int w, int h) { return ssim_impl(a, b, w, h, nullptr); }
double hgso_ssim_with_grad(const double* a, const double* b, int w, int h, double* grad) {
    std::fill(grad, grad + size_t(w) * h * 3, 0.0);
    return ssim_impl(a, b, w, h, grad);
}
double hgso_psnr(const double* a, const double* b, int w, int h) { return psnr(a, b, size_t(w) * h * 3); }

int hgso_optimizer_step(hgso_scene* s, const hgso_grads* g, hgso_state* st, const hgso_lrs* lrs,
                        double mean_lr_scale) {
    return guard([&] { optimizer_step(*s, *g, *st, *lrs, mean_lr_scale); });
}

// train.cpp:433-444
void hgso_accumulate_stats(const hgso_scene* shape, hgso_state* st, const hgso_grads* g) {
    for (int64_t i = 0; i < shape->n3; ++i)
        if (g->screen_norm3[i] > 0.0) {
            st->grad_norm3[i] += g->screen_norm3[i];
            st->count3[i]++;
        }
    for (int64_t i = 0; i < shape->n4; ++i)
        if (g->screen_norm4[i] > 0.0) {
            st->grad_norm4[i] += g->screen_norm4[i];
            st->count4[i]++;
        }
}

int hgso_is_static(double log_st, double tau, int* out) {
    return guard([&] { *out = is_static(log_st, tau) ? 1 : 0; });
}
int hgso_sweep_convert(hgso_scene* s, hgso_state* st, int64_t* moved, hgso_conversion* rep) {
    return guard([&] { sweep_convert(*s, st, moved, *rep); });
}
int hgso_convert_4d_to_3d(const double mean_x[3], double mean_t, const double ql[4], const double qr[4],
                          const double log_s4[4], double op, double mean3[3], double quat3[4],
                          double log_s3[3], double* op3) {
    return guard([&] {
        hgso_scene tmp{};
        tmp.n4 = 1;
        tmp.mean_x = const_cast<double*>(mean_x);
        tmp.mean_t = &mean_t;
        tmp.ql = const_cast<double*>(ql);
        tmp.qr = const_cast<double*>(qr);
        tmp.log_s4 = const_cast<double*>(log_s4);
        tmp.op4 = &op;
        convert_one(tmp, 0, mean3, quat3, log_s3, op3);
    });
}

int hgso_hardware_threads(void) { return int(std::thread::hardware_concurrency()); }

// One training iteration (train.cpp:402-450): per batch image forward_train
// + photometric_loss_with_grad + backward (one std::thread per image when
// num_threads > 1, as the reference does), grads averaged with add_scaled(1/B)
// in index order, raw densify statistics, NumericAbort on a non-finite loss,
// optimizer_step.  The forward uses the tiled tape (bitwise equal to the
// literal forward_train, test_backward.cpp:98-100) with tile_threads.
int hgso_train_step(hgso_scene* s, hgso_state* st, const hgso_camera* cams, const double* times,
                    const double* const* gts, int n_views, const double bg[3], double cutoff, double lambda,
                    const hgso_lrs* lrs, double mean_lr_scale, int num_threads, int tile_threads, double* loss_out) {
    return guard([&] {
        View v{s, sh_count(s->sh_degree)};
        const int K3 = sh_count(s->sh_degree) * 3;
        const int64_t n4 = s->n4, n3 = s->n3;
        struct Buf {
            std::vector<double> d[14];
            hgso_grads g;
        };
        auto alloc = [&](Buf& b) {
            const size_t sz[14] = {size_t(n4 * 3), size_t(n4), size_t(n4 * 4), size_t(n4 * 4), size_t(n4 * 4),
                                   size_t(n4), size_t(n4 * K3), size_t(n4), size_t(n3 * 3), size_t(n3 * 4),
                                   size_t(n3 * 3), size_t(n3), size_t(n3 * K3), size_t(n3)};
            for (int k = 0; k < 14; ++k) b.d[k].assign(sz[k], 0.0);
            double** p = &b.g.mean_x;
            for (int k = 0; k < 14; ++k) p[k] = b.d[k].data();
        };
        std::vector<Buf> per(static_cast<size_t>(n_views));
        std::vector<double> losses(size_t(n_views), 0.0);
        std::vector<std::string> errs(static_cast<size_t>(n_views));
        auto run_one = [&](int bi) {
            try {
                Cam cam = to_cam(cams[bi]);
                const size_t npx = size_t(cam.width) * cam.height;
                std::vector<double> img(npx * 3), lg(npx * 3);
                std::unique_ptr<Tape> tape(forward_train_tiled(v, cam, times[bi], bg, cutoff, tile_threads, img.data()));
                double loss = (1.0 - lambda) * l1(img.data(), gts[bi], npx * 3, lg.data());
                for (double& x : lg) x *= (1.0 - lambda);
                if (lambda != 0.0) {
                    std::vector<double> sg(npx * 3, 0.0);
                    double ss = ssim_impl(img.data(), gts[bi], cam.width, cam.height, sg.data());
                    loss += lambda * (1.0 - ss);
                    for (size_t i = 0; i < lg.size(); ++i) lg[i] -= lambda * sg[i];
                }
                losses[size_t(bi)] = loss;
                alloc(per[size_t(bi)]);
                backward(v, cam, *tape, lg.data(), per[size_t(bi)].g);
            } catch (const std::exception& e) {
                errs[size_t(bi)] = e.what();
            }
        };
        if (num_threads > 1 && n_views > 1) {
            std::vector<std::thread> pool;
            for (int bi = 0; bi < n_views; ++bi) pool.emplace_back(run_one, bi);
            for (auto& th : pool) th.join();
        } else {
            for (int bi = 0; bi < n_views; ++bi) run_one(bi);
        }
        for (const auto& e : errs)
            if (!e.empty()) throw std::invalid_argument(e);
        Buf acc;
        alloc(acc);
        double loss = 0.0;
        for (int bi = 0; bi < n_views; ++bi) {
            loss += losses[size_t(bi)];
            grads_add_scaled(*s, acc.g, per[size_t(bi)].g, 1.0 / double(n_views));
            hgso_accumulate_stats(s, st, &per[size_t(bi)].g);
        }
        loss /= double(n_views);
        if (loss_out) *loss_out = loss;
        if (!std::isfinite(loss)) throw NumericAbort("train: non-finite loss");
        optimizer_step(*s, acc.g, *st, *lrs, mean_lr_scale);
    });
}

}  // extern "C"
