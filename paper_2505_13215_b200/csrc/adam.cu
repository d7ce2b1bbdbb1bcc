// adam.cu -- K8: fused Adam step + gradient zeroing (train.cpp:18-180).
//
// Reference semantics per Gaussian, parameter classes in the reference's
// order (3D: mean, quat, scales, opacity, SH; 4D: mean_x, mean_t, q_left,
// q_right, scales, opacity, SH): skip a whole class if any of its gradients
// is non-finite (counted), else the bias-corrected update with eps = 1e-15;
// quaternions are renormalised every step with the canonical sign and the
// first moment flipped with it (train.cpp:46-53, applied even when the update
// was skipped).
//
// Two passes, both over coalesced SoA rows with float4 (four Gaussians per
// thread; capacities are multiples of 128):
//   adam_classes_kernel  one thread per (class, 4 Gaussians): reads the
//                        class's gradient rows once, writes a finite flag per
//                        (class, Gaussian), fully updates + renormalises the
//                        quaternion classes (their 4 rows belong together),
//                        folds the densification-statistic deltas;
//   adam_rows_kernel     one thread per (row, 4 Gaussians) of every other
//                        row: p, m, v read+write, grad read+zero = 32 B per
//                        element at full memory-level parallelism.  HBM bound.
#include "kernels.cuh"

namespace hgs {

namespace {

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx_a(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }
__device__ __forceinline__ bool fin(float x) { return isfinite(x); }

// One Adam element (train.cpp:155-170); ok = the class is finite.
__device__ __forceinline__ void adam1(float& p, float& m, float& v, float g, bool ok, float lr, const AdamArgs& A) {
    if (!ok) return;
    m = fmaf(A.b1, m, A.one_m_b1 * g);
    v = fmaf(A.b2, v, A.one_m_b2 * g * g);
    const float mhat = m * A.inv_bc1, vhat = v * A.inv_bc2;
    p -= lr * mhat * rcp_approx_a(sqrt_approx(vhat) + 1e-15f);
}

// Parameter class c of a pool: first row, row count, quaternion class.
__device__ __forceinline__ void cls_rows(bool dyn, int c, int K3, int& r0, int& d, bool& quat) {
    quat = false;
    if (dyn) {
        switch (c) {
            case 0: r0 = R4_MEAN, d = 3; break;
            case 1: r0 = R4_MT, d = 1; break;
            case 2: r0 = R4_QL, d = 4, quat = true; break;
            case 3: r0 = R4_QR, d = 4, quat = true; break;
            case 4: r0 = R4_LS, d = 4; break;
            case 5: r0 = R4_OP, d = 1; break;
            default: r0 = R4_SH, d = K3; break;
        }
    } else {
        switch (c) {
            case 0: r0 = R3_MEAN, d = 3; break;
            case 1: r0 = R3_Q, d = 4, quat = true; break;
            case 2: r0 = R3_LS, d = 3; break;
            case 3: r0 = R3_OP, d = 1; break;
            default: r0 = R3_SH, d = K3; break;
        }
    }
}

// train.cpp:46-53 followed by UnitQuat::normalized (gauss_math.cpp:35-44)
__device__ __forceinline__ bool renorm_quat(float q[4], float mq[4]) {
    float n = sqrtf(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    float w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
    const bool flip = w < 0.f || (w == 0.f && (x < 0.f || (x == 0.f && (y < 0.f || (y == 0.f && z < 0.f)))));
    if (flip)
        for (int k = 0; k < 4; ++k) mq[k] = -mq[k];
    n = sqrtf(w * w + x * x + y * y + z * z);
    if (!(n > 0.f) || !isfinite(n)) return false;
    w /= n;
    x /= n;
    y /= n;
    z /= n;
    const float s = flip ? -1.f : 1.f;
    q[0] = s * w;
    q[1] = s * x;
    q[2] = s * y;
    q[3] = s * z;
    return true;
}

// train.cpp:445-447: a non-finite loss aborts the step before the update.
// With pipelined iterations the abort is sticky: every later update is
// skipped too until the host collects the failure.
__device__ __forceinline__ bool update_allowed(const AdamArgs& A) {
    if (A.abort && *(volatile const uint32_t*)A.abort) return false;
    for (int v = 0; v < A.n_views; ++v)
        if (!isfinite(A.view_sums[2 * v]) || !isfinite(A.view_sums[2 * v + 1])) {
            if (A.abort && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.abort, 1u);
            return false;
        }
    return true;
}

}  // namespace

__global__ void __launch_bounds__(128, 6) adam_classes_kernel(AdamPools P, AdamArgs A, uint8_t* __restrict__ cls_ok3,
                                                           uint8_t* __restrict__ cls_ok4,
                                                           unsigned long long* __restrict__ skipped_total,
                                                           uint32_t* __restrict__ flags) {
    pdl_wait();  // launched with launch_pdl
    // one thread per (parameter class, 4 consecutive Gaussians); 3D units
    // first.  The SH class (the bulk of the rows) is checked by adam_sh_slices
    // threads per 4 Gaussians, each over a slice of its rows (slice fastest:
    // a load instruction covers 8 groups x 16 B of 4 rows), flags combined
    // by two shuffles.  Units: 3D classes 0-3 | 3D SH | 4D classes 0-5 |
    // pad to a multiple of 4 | 4D SH.
    if (!update_allowed(A)) return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int S = adam_sh_slices(P.K3);
    const int q3 = (P.n3 + 3) >> 2, q4 = (P.n4 + 3) >> 2;
    const int a3 = 4 * q3, e3 = a3 + S * q3, b4 = e3 + 6 * q4, a4 = e3 + ((6 * q4 + 3) & ~3), e4 = a4 + S * q4;
    bool active = true, dyn = false;
    int c = 0, grp = 0, sl = 0;
    if (t < a3) {
        c = t / q3, grp = t - c * q3;
    } else if (t < e3) {
        c = 4, grp = (t - a3) / S, sl = (t - a3) - grp * S;
    } else if (t < b4) {
        dyn = true, c = (t - e3) / q4, grp = (t - e3) - c * q4;
    } else if (t >= a4 && t < e4) {
        dyn = true, c = 6, grp = (t - a4) / S, sl = (t - a4) - grp * S;
    } else {
        active = false;
    }
    const bool sliced = active && S > 1 && ((!dyn && c == 4) || (dyn && c == 6));
    uint32_t skipped = 0;
    bool ok = true;
    const int i0 = grp * 4;
    const int n = dyn ? P.n4 : P.n3;
    const int64_t cap = dyn ? P.cap4 : P.cap3;
    float* p = dyn ? P.p4 : P.p3;
    float* g = dyn ? P.g4 : P.g3;
    float* m = dyn ? P.m4 : P.m3;
    float* v = dyn ? P.v4 : P.v3;
    int r0 = 0, d = 0;
    bool quat = false;
    cls_rows(dyn, c, P.K3, r0, d, quat);
    uint32_t fm = 0xfu;  // finite flags of the 4 Gaussians (bit w)
    if (active) {
        int k0 = 0, k1 = d;
        if (sliced) {
            const int R = (d + S - 1) / S;
            k0 = min(d, sl * R), k1 = min(d, k0 + R);
        }
        bool f0 = true, f1 = true, f2 = true, f3 = true;
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
            const float4 gv = __ldg(reinterpret_cast<const float4*>(g + (int64_t)(r0 + k) * cap + i0));
            f0 &= fin(gv.x);
            f1 &= fin(gv.y);
            f2 &= fin(gv.z);
            f3 &= fin(gv.w);
        }
        fm = (uint32_t)f0 | ((uint32_t)f1 << 1) | ((uint32_t)f2 << 2) | ((uint32_t)f3 << 3);
    }
    if (S > 1) {  // (every lane: aligned groups of S lanes are one SH group)
        uint32_t x = fm & __shfl_xor_sync(0xffffffffu, fm, 1);
        if (S > 2) x &= __shfl_xor_sync(0xffffffffu, x, 2);
        if (sliced) fm = x;
    }
    if (active && sl == 0) {
        const int nvalid = min(4, n - i0);
        skipped = (uint32_t)__popc(~fm & ((1u << nvalid) - 1u));
        uint8_t* out = (dyn ? cls_ok4 : cls_ok3) + (int64_t)c * cap + i0;
        *reinterpret_cast<uchar4*>(out) = make_uchar4(fm & 1u, (fm >> 1) & 1u, (fm >> 2) & 1u, (fm >> 3) & 1u);
        if (quat) {
            // quaternion class: update, renormalise (even if skipped), zero its
            // gradient; two Gaussians (float2 columns) at a time
#pragma unroll 1
            for (int h = 0; 2 * h < nvalid; ++h) {
                float2 pr[4], mr[4], vr[4], gr[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t o = (int64_t)(r0 + k) * cap + i0 + 2 * h;
                    pr[k] = __ldcs(reinterpret_cast<const float2*>(p + o));
                    mr[k] = __ldcs(reinterpret_cast<const float2*>(m + o));
                    vr[k] = __ldcs(reinterpret_cast<const float2*>(v + o));
                    gr[k] = __ldcs(reinterpret_cast<const float2*>(g + o));
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int w = 2 * h + e;
                    if (w >= nvalid) break;
                    float qv[4], mq[4], vq[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        qv[k] = e ? pr[k].y : pr[k].x;
                        mq[k] = e ? mr[k].y : mr[k].x;
                        vq[k] = e ? vr[k].y : vr[k].x;
                        adam1(qv[k], mq[k], vq[k], e ? gr[k].y : gr[k].x, (fm >> w) & 1u, A.lr_quat, A);
                    }
                    ok &= renorm_quat(qv, mq);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (e) pr[k].y = qv[k], mr[k].y = mq[k], vr[k].y = vq[k];
                        else pr[k].x = qv[k], mr[k].x = mq[k], vr[k].x = vq[k];
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t o = (int64_t)(r0 + k) * cap + i0 + 2 * h;
                    __stcs(reinterpret_cast<float2*>(p + o), pr[k]);
                    __stcs(reinterpret_cast<float2*>(m + o), mr[k]);
                    __stcs(reinterpret_cast<float2*>(v + o), vr[k]);
                    __stcs(reinterpret_cast<float2*>(g + o), make_float2(0.f, 0.f));
                }
            }
        }
        if (c == 0) {
            // fold this step's densification-statistic deltas (train.cpp:433-444)
            float* gn = dyn ? P.gn4 : P.gn3;
            float* cnt = dyn ? P.cnt4 : P.cnt3;
            float* dgn = dyn ? P.dgn4 : P.dgn3;
            float* dcnt = dyn ? P.dcnt4 : P.dcnt3;
            const float4 dg = *reinterpret_cast<const float4*>(dgn + i0);
            const float4 dc = *reinterpret_cast<const float4*>(dcnt + i0);
            if (dg.x != 0.f || dg.y != 0.f || dg.z != 0.f || dg.w != 0.f || dc.x != 0.f || dc.y != 0.f ||
                dc.z != 0.f || dc.w != 0.f) {
                float4 a = *reinterpret_cast<float4*>(gn + i0), b = *reinterpret_cast<float4*>(cnt + i0);
                a.x += dg.x, a.y += dg.y, a.z += dg.z, a.w += dg.w;
                b.x += dc.x, b.y += dc.y, b.z += dc.z, b.w += dc.w;
                *reinterpret_cast<float4*>(gn + i0) = a;
                *reinterpret_cast<float4*>(cnt + i0) = b;
                *reinterpret_cast<float4*>(dgn + i0) = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(dcnt + i0) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    const unsigned full = 0xffffffffu;
    const uint32_t s = __reduce_add_sync(full, skipped);
    if ((threadIdx.x & 31) == 0 && s) {
        atomicAdd(skipped_total, (unsigned long long)s);
        if (A.skipped_cum) atomicAdd(A.skipped_cum, (unsigned long long)s);
    }
    const unsigned bad = __ballot_sync(full, !ok);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, FLAG_NONUNIT_QUAT);
}

// Every non-quaternion row: block b covers 4*blockDim Gaussians of one row.
__global__ void __launch_bounds__(256) adam_rows_kernel(AdamPools P, AdamArgs A, const uint8_t* __restrict__ cls_ok3,
                                                        const uint8_t* __restrict__ cls_ok4, int blocks_per_row3,
                                                        int blocks_per_row4) {
    pdl_wait();  // launched with launch_pdl
    if (!update_allowed(A)) return;
    const int R3 = R3_SH + P.K3 - 4, R4 = R4_SH + P.K3 - 8;  // rows without the quaternions
    int b = blockIdx.x;
    const bool dyn = b >= R3 * blocks_per_row3;
    if (dyn) b -= R3 * blocks_per_row3;
    const int bpr = dyn ? blocks_per_row4 : blocks_per_row3;
    const int rr = b / bpr;  // compacted row index
    if (rr >= (dyn ? R4 : R3)) return;
    const int i0 = ((b % bpr) * blockDim.x + threadIdx.x) * 4;
    const int n = dyn ? P.n4 : P.n3;
    if (i0 >= n) return;
    // compacted row -> pool row, class bit, learning rate (warp-uniform)
    int row, c;
    float lr;
    if (dyn) {
        row = rr < 4 ? rr : rr + 8;  // skip q_left, q_right (rows 4..11)
        if (row < R4_MT) c = 0, lr = A.lr_mean;
        else if (row == R4_MT) c = 1, lr = A.lr_mean_t;
        else if (row < R4_OP) c = 4, lr = A.lr_scales;
        else if (row == R4_OP) c = 5, lr = A.lr_opacity;
        else c = 6, lr = A.lr_sh;
    } else {
        row = rr < 3 ? rr : rr + 4;  // skip the quaternion (rows 3..6)
        if (row < R3_Q) c = 0, lr = A.lr_mean;
        else if (row < R3_OP) c = 2, lr = A.lr_scales;
        else if (row == R3_OP) c = 3, lr = A.lr_opacity;
        else c = 4, lr = A.lr_sh;
    }
    const int64_t o = (int64_t)row * (dyn ? P.cap4 : P.cap3) + i0;
    float* p = (dyn ? P.p4 : P.p3) + o;
    float* g = (dyn ? P.g4 : P.g3) + o;
    float* m = (dyn ? P.m4 : P.m3) + o;
    float* v = (dyn ? P.v4 : P.v3) + o;
    const uchar4 okb =
        *reinterpret_cast<const uchar4*>((dyn ? cls_ok4 : cls_ok3) + (int64_t)c * (dyn ? P.cap4 : P.cap3) + i0);
    float4 pv = ld4(p), gv = ld4(g), mv = ld4(m), vv = ld4(v);
    const int nvalid = min(4, n - i0);
    adam1(pv.x, mv.x, vv.x, gv.x, okb.x, lr, A);
    if (nvalid > 1) adam1(pv.y, mv.y, vv.y, gv.y, okb.y, lr, A);
    if (nvalid > 2) adam1(pv.z, mv.z, vv.z, gv.z, okb.z, lr, A);
    if (nvalid > 3) adam1(pv.w, mv.w, vv.w, gv.w, okb.w, lr, A);
    st4(p, pv);
    st4(m, mv);
    st4(v, vv);
    st4(g, make_float4(0.f, 0.f, 0.f, 0.f));
}

// Packed gradient payload for the multi-GPU all-reduce: the valid part of
// every gradient row ([0, n) of each [row][cap] row) and the two stat-delta
// rows of each pool, contiguous.  Segment s covers pool rows then deltas:
// [g4 rows | g3 rows | dgn4 | dgn3 | dcnt4 | dcnt3].
__global__ void __launch_bounds__(256) grads_pack_kernel(const float* __restrict__ gbuf, int64_t off_g3,
                                                         int64_t off_dgn4, int rows4, int rows3, int64_t cap4,
                                                         int64_t cap3, int n4, int n3, float* __restrict__ packed,
                                                         int unpack) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t a4 = (int64_t)rows4 * n4, a3 = (int64_t)rows3 * n3;
    const int64_t total = a4 + a3 + 2 * (int64_t)n4 + 2 * (int64_t)n3;
    if (e >= total) return;
    int64_t src;
    if (e < a4) {
        src = (e / n4) * cap4 + e % n4;
    } else if (e < a4 + a3) {
        const int64_t k = e - a4;
        src = off_g3 + (k / n3) * cap3 + k % n3;
    } else {
        // delta rows: dgn4 (cap4) | dgn3 (cap3) | dcnt4 (cap4) | dcnt3 (cap3)
        int64_t k = e - a4 - a3;
        int64_t base = off_dgn4;
        if (k < n4) {
            src = base + k;
        } else if ((k -= n4) < n3) {
            src = base + cap4 + k;
        } else if ((k -= n3) < n4) {
            src = base + cap4 + cap3 + k;
        } else {
            k -= n4;
            src = base + 2 * cap4 + cap3 + k;
        }
    }
    if (unpack) const_cast<float*>(gbuf)[src] = packed[e];
    else packed[e] = gbuf[src];
}

}  // namespace hgs
