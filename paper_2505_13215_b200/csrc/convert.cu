// convert.cu -- K9: tau-threshold 4D->3D conversion as stream compaction
// (scene.cpp:10-71 sweep_convert + train.cpp:305-362 remap_after_sweep).
//
//  mask     : exp(s_t) > tau  <=>  (double)s_t >= s_star, with s_star the
//             smallest double for which the host libm exp exceeds tau
//             (computed once per sweep on the host), so the predicate is
//             bit-exact against the reference for every input;
//  scan     : exclusive scan of the mask -> converted slot k / survivor slot;
//  convert  : one thread per converted row: polar factor of R4[0:3,0:3]
//             (one-sided Jacobi SVD, FP64) -> quaternion, opacity folded by
//             the erf mean temporal weight, SH copied; Adam rows inherit
//             mean_x, scales[0:3], q_left, opacity, SH moments;
//  compact  : survivors (params, m, v) gathered stably into the alternate
//             buffers, which are then swapped in.
#include "kernels.cuh"

namespace hgs {

namespace {

struct M3 {
    double a[3][3];
};

__device__ inline double det3(const M3& m) {
    const auto& a = m.a;
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

// One-sided Jacobi SVD (same algorithm as the oracle's svd3).
__device__ void svd3(const M3& a, M3& u, double sv[3], M3& v) {
    M3 b = a;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v.a[i][j] = i == j ? 1.0 : 0.0;
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
                if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
                changed = true;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int k = 0; k < 3; ++k) {
                    const double bp = b.a[k][p], bq = b.a[k][q];
                    b.a[k][p] = c * bp - s * bq;
                    b.a[k][q] = s * bp + c * bq;
                    const double vp = v.a[k][p], vq = v.a[k][q];
                    v.a[k][p] = c * vp - s * vq;
                    v.a[k][q] = s * vp + c * vq;
                }
            }
        if (!changed) break;
    }
    double n[3];
    for (int c = 0; c < 3; ++c) n[c] = sqrt(b.a[0][c] * b.a[0][c] + b.a[1][c] * b.a[1][c] + b.a[2][c] * b.a[2][c]);
    int idx[3] = {0, 1, 2};
    for (int i = 1; i < 3; ++i)
        for (int j = i; j > 0 && n[idx[j]] > n[idx[j - 1]]; --j) {
            const int tmp = idx[j];
            idx[j] = idx[j - 1];
            idx[j - 1] = tmp;
        }
    M3 bs, vs;
    for (int c = 0; c < 3; ++c) {
        sv[c] = n[idx[c]];
        for (int r = 0; r < 3; ++r) {
            bs.a[r][c] = b.a[r][idx[c]];
            vs.a[r][c] = v.a[r][idx[c]];
        }
    }
    v = vs;
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) u.a[r][c] = sv[c] > 1e-300 ? bs.a[r][c] / sv[c] : 0.0;
    if (sv[2] <= 1e-15 * fmax(sv[0], 1e-300)) {
        u.a[0][2] = u.a[1][0] * u.a[2][1] - u.a[2][0] * u.a[1][1];
        u.a[1][2] = u.a[2][0] * u.a[0][1] - u.a[0][0] * u.a[2][1];
        u.a[2][2] = u.a[0][0] * u.a[1][1] - u.a[1][0] * u.a[0][1];
    }
}

__device__ inline M3 mul3T(const M3& x, const M3& y) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r.a[i][j] = x.a[i][0] * y.a[j][0] + x.a[i][1] * y.a[j][1] + x.a[i][2] * y.a[j][2];
    return r;
}

__device__ inline bool is_rotation(const M3& m, double tol) {
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const double s = m.a[0][i] * m.a[0][j] + m.a[1][i] * m.a[1][j] + m.a[2][i] * m.a[2][j];
            worst = fmax(worst, fabs(s - (i == j ? 1.0 : 0.0)));
        }
    return worst <= tol && fabs(det3(m) - 1.0) <= tol;
}

// gauss_math.cpp:70-97 (+ UnitQuat::normalized)
__device__ inline bool rot3_to_quat(const M3& m, double q[4]) {
    if (!is_rotation(m, 1e-6)) return false;
    const auto& r = m.a;
    const double tr = r[0][0] + r[1][1] + r[2][2];
    double w, x, y, z;
    if (1.0 + tr >= 1e-6) {
        w = 0.5 * sqrt(1.0 + tr);
        x = (r[2][1] - r[1][2]) / (4.0 * w);
        y = (r[0][2] - r[2][0]) / (4.0 * w);
        z = (r[1][0] - r[0][1]) / (4.0 * w);
    } else {
        int i = 0;
        if (r[1][1] > r[0][0]) i = 1;
        if (r[2][2] > r[i][i]) i = 2;
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        const double s = sqrt(r[i][i] - r[j][j] - r[k][k] + 1.0);
        double vv[3];
        vv[i] = 0.5 * s;
        const double inv = 0.5 / s;
        w = (r[k][j] - r[j][k]) * inv;
        vv[j] = (r[j][i] + r[i][j]) * inv;
        vv[k] = (r[k][i] + r[i][k]) * inv;
        x = vv[0];
        y = vv[1];
        z = vv[2];
    }
    const double n = sqrt(w * w + x * x + y * y + z * z);
    w /= n;
    x /= n;
    y /= n;
    z /= n;
    bool flip = false;
    if (w < 0.0) flip = true;
    else if (w == 0.0) flip = x != 0.0 ? x < 0.0 : (y != 0.0 ? y < 0.0 : z < 0.0);
    if (flip) {
        w = -w;
        x = -x;
        y = -y;
        z = -z;
    }
    q[0] = w;
    q[1] = x;
    q[2] = y;
    q[3] = z;
    return true;
}

__device__ inline double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

// scene.cpp:19-31
__device__ inline double fold_temporal_weight(double op, double mean_t, double sigma_t) {
    const double s = sigma_t * sqrt(2.0);
    double w = sigma_t * sqrt(M_PI / 2.0) * (erf((1.0 - mean_t) / s) + erf(mean_t / s));
    w = w < 1.0 ? w : 1.0;
    if (w >= 1.0 - 1e-12) return op;
    const double alpha = sigmoid(op) * w;
    return log(alpha) - log1p(-alpha);
}

}  // namespace

__global__ void __launch_bounds__(256) convert_mask_kernel(const float* __restrict__ p4, int64_t cap4, int n4,
                                                           double s_star, uint32_t* __restrict__ mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n4) mask[i] = ((double)p4[(int64_t)(R4_LS + 3) * cap4 + i] >= s_star) ? 1u : 0u;
}

// Converted rows: append to the 3D pool at n3 + k (param + Adam moments).
__global__ void __launch_bounds__(128) convert_rows_kernel(
    const float* __restrict__ p4, const float* __restrict__ m4, const float* __restrict__ v4, int64_t cap4, int n4,
    const uint32_t* __restrict__ mask, const uint32_t* __restrict__ pos, float* __restrict__ p3, float* __restrict__ m3,
    float* __restrict__ v3, int64_t cap3, int n3, int deg, long long* __restrict__ moved,
    unsigned long long* __restrict__ max_leak_bits, double* __restrict__ leak_sum, uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4 || !mask[i]) return;
    const uint32_t k = pos[i];
    const int dst = n3 + (int)k;
    if (moved) moved[k] = i;
    auto P = [&](int row) { return (double)p4[(int64_t)row * cap4 + i]; };
    double ql[4], qr[4];
    for (int c = 0; c < 4; ++c) {
        ql[c] = P(R4_QL + c);
        qr[c] = P(R4_QR + c);
    }
    // R4 = L(ql) R(qr); only the 3x3 block and the mixing entries are needed
    const double a = ql[0], b = ql[1], c_ = ql[2], d = ql[3];
    const double L[4][4] = {{a, -b, -c_, -d}, {b, a, -d, c_}, {c_, d, a, -b}, {d, -c_, b, a}};
    const double p = qr[0], q = qr[1], r = qr[2], s = qr[3];
    const double R[4][4] = {{p, -q, -r, -s}, {q, p, s, -r}, {r, -s, p, q}, {s, r, -q, p}};
    double R4[4][4];
    for (int x = 0; x < 4; ++x)
        for (int y = 0; y < 4; ++y) {
            double acc = L[x][0] * R[0][y];
            acc = acc + L[x][1] * R[1][y];
            acc = acc + L[x][2] * R[2][y];
            acc = acc + L[x][3] * R[3][y];
            R4[x][y] = acc;
        }
    M3 block, u, v;
    for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y) block.a[x][y] = R4[x][y];
    double sv[3];
    svd3(block, u, sv, v);
    if (sv[0] < 1e-9) atomicOr(flags, FLAG_DEGENERATE_ROT);
    if (det3(mul3T(u, v)) < 0.0)
        for (int x = 0; x < 3; ++x) u.a[x][2] = -u.a[x][2];
    const M3 rot = mul3T(u, v);
    double quat[4];
    if (!rot3_to_quat(rot, quat)) atomicOr(flags, FLAG_NOT_ROTATION);
    const double leak = sqrt(R4[0][3] * R4[0][3] + R4[1][3] * R4[1][3] + R4[2][3] * R4[2][3] + R4[3][0] * R4[3][0] +
                             R4[3][1] * R4[3][1] + R4[3][2] * R4[3][2]);
    atomicMax(max_leak_bits, (unsigned long long)__double_as_longlong(leak));
    atomicAdd(leak_sum, leak);
    auto W3 = [&](float* buf, int row, float val) { buf[(int64_t)row * cap3 + dst] = val; };
    for (int c = 0; c < 3; ++c) W3(p3, R3_MEAN + c, (float)P(R4_MEAN + c));
    for (int c = 0; c < 4; ++c) W3(p3, R3_Q + c, (float)quat[c]);
    for (int c = 0; c < 3; ++c) W3(p3, R3_LS + c, (float)P(R4_LS + c));
    W3(p3, R3_OP, (float)fold_temporal_weight(P(R4_OP), P(R4_MT), exp(P(R4_LS + 3))));
    const int K3 = 3 * sh_count(deg);
    for (int c = 0; c < K3; ++c) W3(p3, R3_SH + c, p4[(int64_t)(R4_SH + c) * cap4 + i]);
    // train.cpp:323-341: moment inheritance
    for (int pass = 0; pass < 2; ++pass) {
        const float* S = pass ? v4 : m4;
        float* D = pass ? v3 : m3;
        auto cp = [&](int drow, int srow) { D[(int64_t)drow * cap3 + dst] = S[(int64_t)srow * cap4 + i]; };
        for (int c = 0; c < 3; ++c) cp(R3_MEAN + c, R4_MEAN + c);
        for (int c = 0; c < 3; ++c) cp(R3_LS + c, R4_LS + c);
        for (int c = 0; c < 4; ++c) cp(R3_Q + c, R4_QL + c);
        cp(R3_OP, R4_OP);
        for (int c = 0; c < K3; ++c) cp(R3_SH + c, R4_SH + c);
    }
}

// Stable compaction of the surviving 4D rows into the alternate buffers.
__global__ void __launch_bounds__(256) compact_survivors_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                                int rows, int64_t cap4, int n4,
                                                                const uint32_t* __restrict__ mask,
                                                                const uint32_t* __restrict__ pos) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4 || mask[i]) return;
    const int o = i - (int)pos[i];
    for (int r = 0; r < rows; ++r) dst[(int64_t)r * cap4 + o] = src[(int64_t)r * cap4 + i];
}

}  // namespace hgs
