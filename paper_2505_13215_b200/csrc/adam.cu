// adam.cu -- K8: fused Adam step + gradient zeroing (train.cpp:18-180).
//
// One thread per Gaussian row, looping over the parameter classes in the
// reference's order (3D: mean, quat, scales, opacity, SH; 4D: mean_x, mean_t,
// q_left, q_right, scales, opacity, SH).  Per row and class: skip the whole
// class if any gradient is non-finite (counted), else the bias-corrected
// update with eps = 1e-15; quaternions are renormalised every step with the
// canonical sign and the first moment flipped with it (train.cpp:46-53,
// applied even when the update was skipped).  Every component access is a
// coalesced SoA row; the gradient is zeroed in the same pass.
// Bytes per element: param, m, v read+write, grad read+zero = 32 B.  HBM bound.
#include "kernels.cuh"

namespace hgs {


namespace {

__device__ __forceinline__ bool row_finite(const float* g, int64_t cap, int i, int r0, int d) {
    bool ok = true;
#pragma unroll 8
    for (int k = 0; k < d; ++k) ok &= isfinite(g[(int64_t)(r0 + k) * cap + i]);
    return ok;
}

__device__ __forceinline__ void adam_class(float* p, float* g, float* m, float* v, int64_t cap, int i, int r0, int d,
                                           float lr, const AdamArgs& A, uint32_t& skipped) {
    if (!row_finite(g, cap, i, r0, d)) {
        ++skipped;
        for (int k = 0; k < d; ++k) g[(int64_t)(r0 + k) * cap + i] = 0.f;
        return;
    }
    // chunks of 8 rows: all 32 loads of a chunk are issued before any store
    // (memory-level parallelism; the four arrays never alias)
    constexpr int C = 8;
    for (int k0 = 0; k0 < d; k0 += C) {
        float gr[C], mm[C], vv[C], pp[C];
#pragma unroll
        for (int u = 0; u < C; ++u) {
            if (k0 + u < d) {
                const int64_t o = (int64_t)(r0 + k0 + u) * cap + i;
                gr[u] = __ldcs(&g[o]);
                mm[u] = __ldcs(&m[o]);
                vv[u] = __ldcs(&v[o]);
                pp[u] = __ldcs(&p[o]);
            }
        }
#pragma unroll
        for (int u = 0; u < C; ++u) {
            if (k0 + u < d) {
                const int64_t o = (int64_t)(r0 + k0 + u) * cap + i;
                const float mk = A.b1 * mm[u] + A.one_m_b1 * gr[u];
                const float vk = A.b2 * vv[u] + A.one_m_b2 * gr[u] * gr[u];
                const float mhat = mk * A.inv_bc1, vhat = vk * A.inv_bc2;
                __stcs(&m[o], mk);
                __stcs(&v[o], vk);
                __stcs(&p[o], pp[u] - lr * mhat / (sqrtf(vhat) + 1e-15f));
                __stcs(&g[o], 0.f);
            }
        }
    }
}

// train.cpp:46-53 followed by UnitQuat::normalized (gauss_math.cpp:35-44)
__device__ __forceinline__ bool renorm_quat(float* p, float* m, int64_t cap, int i, int r0) {
    float q[4];
    for (int k = 0; k < 4; ++k) q[k] = p[(int64_t)(r0 + k) * cap + i];
    float n = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    const bool flip = w < 0.f || (w == 0.f && (x < 0.f || (x == 0.f && (y < 0.f || (y == 0.f && z < 0.f)))));
    if (flip)
        for (int k = 0; k < 4; ++k) m[(int64_t)(r0 + k) * cap + i] = -m[(int64_t)(r0 + k) * cap + i];
    n = sqrtf(w * w + x * x + y * y + z * z);
    if (!(n > 0.f) || !isfinite(n)) return false;
    w /= n;
    x /= n;
    y /= n;
    z /= n;
    if (flip) {
        w = -w;
        x = -x;
        y = -y;
        z = -z;
    }
    p[(int64_t)(r0 + 0) * cap + i] = w;
    p[(int64_t)(r0 + 1) * cap + i] = x;
    p[(int64_t)(r0 + 2) * cap + i] = y;
    p[(int64_t)(r0 + 3) * cap + i] = z;
    return true;
}

}  // namespace

__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p4, float* __restrict__ g4, float* __restrict__ m4,
                                                   float* __restrict__ v4, int64_t cap4, int n4, float* __restrict__ p3,
                                                   float* __restrict__ g3, float* __restrict__ m3, float* __restrict__ v3,
                                                   int64_t cap3, int n3, int deg, AdamArgs A,
                                                   unsigned long long* __restrict__ skipped_total,
                                                   uint32_t* __restrict__ flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t skipped = 0;
    bool ok = true;
    const int K3 = 3 * sh_count(deg);
    if (t < n3) {
        const int i = t;
        adam_class(p3, g3, m3, v3, cap3, i, R3_MEAN, 3, A.lr_mean, A, skipped);
        adam_class(p3, g3, m3, v3, cap3, i, R3_Q, 4, A.lr_quat, A, skipped);
        ok &= renorm_quat(p3, m3, cap3, i, R3_Q);
        adam_class(p3, g3, m3, v3, cap3, i, R3_LS, 3, A.lr_scales, A, skipped);
        adam_class(p3, g3, m3, v3, cap3, i, R3_OP, 1, A.lr_opacity, A, skipped);
        adam_class(p3, g3, m3, v3, cap3, i, R3_SH, K3, A.lr_sh, A, skipped);
    } else if (t < n3 + n4) {
        const int i = t - n3;
        adam_class(p4, g4, m4, v4, cap4, i, R4_MEAN, 3, A.lr_mean, A, skipped);
        adam_class(p4, g4, m4, v4, cap4, i, R4_MT, 1, A.lr_mean_t, A, skipped);
        adam_class(p4, g4, m4, v4, cap4, i, R4_QL, 4, A.lr_quat, A, skipped);
        ok &= renorm_quat(p4, m4, cap4, i, R4_QL);
        adam_class(p4, g4, m4, v4, cap4, i, R4_QR, 4, A.lr_quat, A, skipped);
        ok &= renorm_quat(p4, m4, cap4, i, R4_QR);
        adam_class(p4, g4, m4, v4, cap4, i, R4_LS, 4, A.lr_scales, A, skipped);
        adam_class(p4, g4, m4, v4, cap4, i, R4_OP, 1, A.lr_opacity, A, skipped);
        adam_class(p4, g4, m4, v4, cap4, i, R4_SH, K3, A.lr_sh, A, skipped);
    }
    const unsigned full = 0xffffffffu;
    const uint32_t s = __reduce_add_sync(full, skipped);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(skipped_total, (unsigned long long)s);
    const unsigned bad = __ballot_sync(full, !ok);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, FLAG_NONUNIT_QUAT);
}

// Fold this step's densify-statistic deltas into the running sums
// (train.cpp:433-444) and clear them.
__global__ void __launch_bounds__(256) fold_stats_kernel(float* __restrict__ gn, float* __restrict__ cnt,
                                                         float* __restrict__ dgn, float* __restrict__ dcnt, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float d = dgn[i], c = dcnt[i];
    if (c != 0.f || d != 0.f) {
        gn[i] += d;
        cnt[i] += c;
        dgn[i] = 0.f;
        dcnt[i] = 0.f;
    }
}

}  // namespace hgs
