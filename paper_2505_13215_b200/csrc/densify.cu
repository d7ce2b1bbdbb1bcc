// densify.cu -- densify_and_prune on the device (train.cpp:182-299, SURVEY.md
// 8f-1), the periodic step of the training loop that changes the pool sizes.
//
// Plan (hgs_densify_plan): per pool, one thread per Gaussian classifies it
// (prune if sigmoid(opacity) < eps; a densification candidate if the averaged
// screen gradient exceeds the threshold -- clone when the largest spatial
// scale is below clone_size_frac * extent, else split).  The reference's
// sequential capacity rule `out.size() + 2 <= max_gaussians` only ever stops
// densifying from one candidate on (the output size never decreases), so it
// is resolved with a scan assuming every candidate densifies, the first
// candidate that would overflow (atomicMin), a downgrade of the candidates
// from there on, and a second scan for the output positions.  The ordered
// list of densified Gaussians (1 = clone, 2 = split) goes back to the host,
// which draws the reference's normal variates in that order.
// Apply (hgs_densify_apply): one thread per source Gaussian writes its 0, 1
// or 2 output rows into freshly allocated pools (SoA, new capacities):
// parameters, and the Adam moments of kept rows (fresh rows start at zero,
// remap_buf train.cpp:56-66); the jitter (R diag(e^s)) n is formed in FP64
// with the oracle's operation order.  Statistics and gradients restart at 0.
#include <algorithm>
#include <cstring>
#include <string>

#include "ctx.cuh"
#include "gauss_math.cuh"
#include "kernels.cuh"
#include "primitives.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

hgs_status fail(hgs_ctx* ctx, hgs_status s, const std::string& m) {
    if (ctx) ctx->err = m;
    return s;
}
#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess)                                                               \
            return fail(ctx, HGS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define CKL() CK(cudaGetLastError())

struct DensifyParams {
    double grad_threshold, opacity_prune_eps, size_gate, log_split;
    int64_t max_gaussians;
};

__global__ void __launch_bounds__(256) densify_classify_kernel(const float* __restrict__ P, int64_t cap, int n, int dyn,
                                                               const float* __restrict__ gn,
                                                               const float* __restrict__ cnt, DensifyParams dp,
                                                               uint8_t* __restrict__ cat, uint32_t* __restrict__ sz) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r_op = dyn ? R4_OP : R3_OP, r_ls = dyn ? R4_LS : R3_LS;
    const double op = P[(int64_t)r_op * cap + i];
    uint8_t c;
    if (1.0 / (1.0 + exp(-op)) < dp.opacity_prune_eps) {
        c = 0;  // pruned
    } else {
        const double k = cnt[i];
        const double avg = k > 0.0 ? (double)gn[i] / k : 0.0;
        if (avg > dp.grad_threshold) {
            const double e0 = exp((double)P[(int64_t)(r_ls + 0) * cap + i]);
            const double e1 = exp((double)P[(int64_t)(r_ls + 1) * cap + i]);
            const double e2 = exp((double)P[(int64_t)(r_ls + 2) * cap + i]);
            c = fmax(fmax(e0, e1), e2) < dp.size_gate ? 2 : 3;  // clone : split
        } else {
            c = 1;
        }
    }
    cat[i] = c;
    sz[i] = c == 0 ? 0u : (c == 1 ? 1u : 2u);
}

// candidates whose output position (every earlier candidate densified) leaves
// no room for two rows
__global__ void __launch_bounds__(256) densify_cap_kernel(const uint8_t* __restrict__ cat,
                                                          const uint32_t* __restrict__ pre, int n, int64_t maxg,
                                                          int* __restrict__ first_bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || cat[i] < 2) return;
    if ((int64_t)pre[i] + 2 > maxg) atomicMin(first_bad, i);
}

__global__ void __launch_bounds__(256) densify_finalize_kernel(uint8_t* __restrict__ cat, int n,
                                                               const int* __restrict__ first_bad,
                                                               uint32_t* __restrict__ sz, uint32_t* __restrict__ dflag,
                                                               unsigned long long* __restrict__ counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t c = cat[i];
    if (c >= 2 && i >= *first_bad) c = 1;  // the reference stops densifying from here on
    cat[i] = c;
    sz[i] = c == 0 ? 0u : (c == 1 ? 1u : 2u);
    dflag[i] = c >= 2 ? 1u : 0u;
    // counts: [0] pruned, [1] cloned, [2] split
    const unsigned full = __activemask();
    const unsigned pm = __ballot_sync(full, c == 0), cm = __ballot_sync(full, c == 2), sm = __ballot_sync(full, c == 3);
    if ((threadIdx.x & 31) == __ffs(full) - 1) {
        if (pm) atomicAdd(&counts[0], (unsigned long long)__popc(pm));
        if (cm) atomicAdd(&counts[1], (unsigned long long)__popc(cm));
        if (sm) atomicAdd(&counts[2], (unsigned long long)__popc(sm));
    }
}

__global__ void __launch_bounds__(256) densify_kinds_kernel(const uint8_t* __restrict__ cat,
                                                            const uint32_t* __restrict__ drank, int n,
                                                            uint8_t* __restrict__ kinds) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && cat[i] >= 2) kinds[drank[i]] = cat[i] - 1;  // 1 clone, 2 split
}

// One source Gaussian -> its output rows.  jit: per densified Gaussian (rank
// order) `stride` doubles: the normal vector(s) n (statics 3 per row, dynamics
// 4 per row; a clone uses the first).
__global__ void __launch_bounds__(128) densify_apply_kernel(const float* __restrict__ Ps, const float* __restrict__ Ms,
                                                            const float* __restrict__ Vs, int64_t caps,
                                                            float* __restrict__ Pd, float* __restrict__ Md,
                                                            float* __restrict__ Vd, int64_t capd, int n, int dyn,
                                                            int rows, const uint8_t* __restrict__ cat,
                                                            const uint32_t* __restrict__ pos,
                                                            const uint32_t* __restrict__ drank,
                                                            const double* __restrict__ jit, double log_split) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t c = cat[i];
    if (c == 0) return;
    const int64_t o = pos[i];
    auto copy_row = [&](int64_t d, bool adam) {
        for (int r = 0; r < rows; ++r) {
            Pd[(int64_t)r * capd + d] = Ps[(int64_t)r * caps + i];
            Md[(int64_t)r * capd + d] = adam ? Ms[(int64_t)r * caps + i] : 0.0f;
            Vd[(int64_t)r * capd + d] = adam ? Vs[(int64_t)r * caps + i] : 0.0f;
        }
    };
    if (c == 1) {
        copy_row(o, true);
        return;
    }
    const int dim = dyn ? 4 : 3;
    const int r_mean = dyn ? R4_MEAN : R3_MEAN, r_ls = dyn ? R4_LS : R3_LS;
    double m[4][4];
    double ls[4];
    for (int b = 0; b < dim; ++b) ls[b] = Ps[(int64_t)(r_ls + b) * caps + i];
    if (dyn) {
        double ql[4], qr[4];
        for (int k = 0; k < 4; ++k) {
            ql[k] = Ps[(int64_t)(R4_QL + k) * caps + i];
            qr[k] = Ps[(int64_t)(R4_QR + k) * caps + i];
        }
        const gm::M4 R = gm::rot4_from_pair(ql, qr);
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) m[a][b] = R.a[a][b] * exp(ls[b]);
    } else {
        double q[4];
        for (int k = 0; k < 4; ++k) q[k] = Ps[(int64_t)(R3_Q + k) * caps + i];
        gm::M3 R;
        gm::quat_to_rot3(q, R);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) m[a][b] = R.a[a][b] * exp(ls[b]);
    }
    const int stride = dyn ? 8 : 6;
    const double* nv = jit + (int64_t)drank[i] * stride;
    auto jitter = [&](const double* nn, double y[4]) {
        for (int a = 0; a < dim; ++a) {
            double s = m[a][0] * nn[0];
            for (int b = 1; b < dim; ++b) s = s + m[a][b] * nn[b];
            y[a] = s;
        }
    };
    if (c == 2) {  // clone: the original (with its moments) + a jittered copy
        copy_row(o, true);
        copy_row(o + 1, false);
        double y[4];
        jitter(nv, y);
        for (int a = 0; a < 3; ++a)
            Pd[(int64_t)(r_mean + a) * capd + o + 1] = (float)((double)Ps[(int64_t)(r_mean + a) * caps + i] + 0.1 * y[a]);
    } else {  // split: two offset parts with smaller scales
        for (int h = 0; h < 2; ++h) {
            copy_row(o + h, false);
            double y[4];
            jitter(nv + h * dim, y);
            for (int a = 0; a < 3; ++a)
                Pd[(int64_t)(r_mean + a) * capd + o + h] = (float)((double)Ps[(int64_t)(r_mean + a) * caps + i] + y[a]);
            if (dyn) Pd[(int64_t)R4_MT * capd + o + h] = (float)((double)Ps[(int64_t)R4_MT * caps + i] + y[3]);
            for (int a = 0; a < dim; ++a) Pd[(int64_t)(r_ls + a) * capd + o + h] = (float)(ls[a] - log_split);
        }
    }
}

int64_t round_cap_d(int64_t n) { return ((n + 127) / 128) * 128 + 128; }

// train.cpp:459-465: opacity logits capped at logit(0.01)
__global__ void opacity_cap_kernel(float* __restrict__ p, int64_t cap, int row, int n, float cap_logit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        float* o = p + (int64_t)row * cap + i;
        *o = fminf(*o, cap_logit);
    }
}


}  // namespace

extern "C" {

hgs_status hgs_densify_plan(hgs_ctx* ctx, const hgs_densify_cfg* cfg, uint8_t* kinds3, uint8_t* kinds4,
                            hgs_densify_report* rep) {
    if (!ctx || !cfg || !rep) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->pipeline.empty()) return fail(ctx, HGS_ERR_STATE, "densify: pipelined iterations pending");
    if (ctx->state_sharded) return fail(ctx, HGS_ERR_STATE, "densify: the Adam moments are sharded (hgs_gather_state on every rank first)");

    if (!(cfg->split_factor > 0.0) || cfg->max_gaussians < 0)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "densify: bad configuration");
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    DensifyParams dp{cfg->grad_threshold, cfg->opacity_prune_eps, cfg->clone_size_frac * ctx->extent,
                     std::log(cfg->split_factor), cfg->max_gaussians};
    const int64_t N = std::max<int64_t>(ctx->n3 + ctx->n4, 1);
    CK(ctx->dens_cat.ensure((size_t)N));
    CK(ctx->dens_u32.ensure((size_t)N * 4 * 5 + 64));
    CK(ctx->dens_misc.ensure(256));
    CK(ctx->scan_ws.ensure(scan_workspace_bytes((int)N) + 4096));
    *rep = hgs_densify_report{};
    uint32_t* base = ctx->dens_u32.as<uint32_t>();
    struct Misc {
        unsigned long long counts[2][3];
        int first_bad[2];
        uint32_t totals[2][2];  // new size, densified count
    };
    Misc* dm = ctx->dens_misc.as<Misc>();
    CK(cudaMemsetAsync(dm, 0, sizeof(Misc), st));
    CK(cudaMemsetAsync(dm->first_bad, 0x7f, sizeof(dm->first_bad), st));
    // statics first, then dynamics (train.cpp:189-298)
    for (int pool = 0; pool < 2; ++pool) {
        const bool dyn = pool == 1;
        const int n = (int)(dyn ? ctx->n4 : ctx->n3);
        const int64_t off = dyn ? ctx->n3 : 0;
        uint8_t* cat = ctx->dens_cat.as<uint8_t>() + off;
        uint32_t* sz = base + off;
        uint32_t* pre = base + N + off;
        uint32_t* dflag = base + 2 * N + off;
        uint32_t* drank = base + 3 * N + off;
        uint32_t* posv = base + 4 * N + off;
        if (n == 0) continue;
        const unsigned g = (unsigned)((n + 255) / 256);
        densify_classify_kernel<<<g, 256, 0, st>>>(dyn ? ctx->p4.as<float>() : ctx->p3.as<float>(),
                                                   dyn ? ctx->cap4 : ctx->cap3, n, dyn ? 1 : 0,
                                                   dyn ? ctx->gn4.as<float>() : ctx->gn3.as<float>(),
                                                   dyn ? ctx->cnt4.as<float>() : ctx->cnt3.as<float>(), dp, cat, sz);
        count_launch();
        CKL();
        exclusive_scan_u32(sz, pre, n, nullptr, ctx->scan_ws.as<uint32_t>(), st);
        densify_cap_kernel<<<g, 256, 0, st>>>(cat, pre, n, cfg->max_gaussians, &dm->first_bad[pool]);
        count_launch();
        densify_finalize_kernel<<<g, 256, 0, st>>>(cat, n, &dm->first_bad[pool], sz, dflag, dm->counts[pool]);
        count_launch();
        exclusive_scan_u32(sz, posv, n, &dm->totals[pool][0], ctx->scan_ws.as<uint32_t>(), st);
        exclusive_scan_u32(dflag, drank, n, &dm->totals[pool][1], ctx->scan_ws.as<uint32_t>(), st);
        CK(ctx->dens_kinds.ensure((size_t)N + 64));
        densify_kinds_kernel<<<g, 256, 0, st>>>(cat, drank, n, ctx->dens_kinds.as<uint8_t>() + off);
        count_launch();
        CKL();
    }
    Misc h;
    CK(cudaMemcpyAsync(&h, dm, sizeof(Misc), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rep->pruned3 = (int64_t)h.counts[0][0];
    rep->cloned3 = (int64_t)h.counts[0][1];
    rep->split3 = (int64_t)h.counts[0][2];
    rep->pruned4 = (int64_t)h.counts[1][0];
    rep->cloned4 = (int64_t)h.counts[1][1];
    rep->split4 = (int64_t)h.counts[1][2];
    ctx->dens_new[0] = ctx->n3 ? h.totals[0][0] : 0;
    ctx->dens_new[1] = ctx->n4 ? h.totals[1][0] : 0;
    ctx->dens_count[0] = ctx->n3 ? h.totals[0][1] : 0;
    ctx->dens_count[1] = ctx->n4 ? h.totals[1][1] : 0;
    rep->new_n3 = ctx->dens_new[0];
    rep->new_n4 = ctx->dens_new[1];
    if (kinds3 && ctx->dens_count[0])
        CK(cudaMemcpy(kinds3, ctx->dens_kinds.as<uint8_t>(), ctx->dens_count[0], cudaMemcpyDeviceToHost));
    if (kinds4 && ctx->dens_count[1])
        CK(cudaMemcpy(kinds4, ctx->dens_kinds.as<uint8_t>() + ctx->n3, ctx->dens_count[1], cudaMemcpyDeviceToHost));
    ctx->dens_planned = true;
    return HGS_OK;
}

hgs_status hgs_densify_apply(hgs_ctx* ctx, const double* normals3, const double* normals4, double split_factor) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->dens_planned) return fail(ctx, HGS_ERR_STATE, "densify_apply: no plan (hgs_densify_plan first)");
    if ((ctx->dens_count[0] && !normals3) || (ctx->dens_count[1] && !normals4) || !(split_factor > 0.0))
        return HGS_ERR_INVALID_ARGUMENT;
    ctx->dens_planned = false;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t st = ctx->stream;
    const int64_t n3 = ctx->n3, n4 = ctx->n4, N = std::max<int64_t>(n3 + n4, 1);
    const int64_t nn3 = ctx->dens_new[0], nn4 = ctx->dens_new[1];
    const int64_t cap4 = round_cap_d(nn4), cap3 = round_cap_d(nn3 + nn4);
    const int r4 = rows4(ctx->deg), r3 = rows3(ctx->deg);
    // the variates, in rank order (stride 6 statics, 8 dynamics)
    const size_t j3 = (size_t)ctx->dens_count[0] * 6, j4 = (size_t)ctx->dens_count[1] * 8;
    CK(ctx->dens_jit.ensure((j3 + j4 + 8) * sizeof(double)));
    double* jit3 = ctx->dens_jit.as<double>();
    double* jit4 = jit3 + j3;
    if (j3) CK(cudaMemcpyAsync(jit3, normals3, j3 * sizeof(double), cudaMemcpyHostToDevice, st));
    if (j4) CK(cudaMemcpyAsync(jit4, normals4, j4 * sizeof(double), cudaMemcpyHostToDevice, st));
    DBuf np4, nm4, nv4, np3, nm3, nv3;
    for (DBuf* b : {&np4, &nm4, &nv4}) CK(b->ensure((size_t)r4 * cap4 * 4));
    for (DBuf* b : {&np3, &nm3, &nv3}) CK(b->ensure((size_t)r3 * cap3 * 4));
    for (DBuf* b : {&np3, &nm3, &nv3}) CK(cudaMemsetAsync(b->p, 0, (size_t)r3 * cap3 * 4, st));
    for (DBuf* b : {&np4, &nm4, &nv4}) CK(cudaMemsetAsync(b->p, 0, (size_t)r4 * cap4 * 4, st));
    uint32_t* base = ctx->dens_u32.as<uint32_t>();
    const double log_split = std::log(split_factor);
    for (int pool = 0; pool < 2; ++pool) {
        const bool dyn = pool == 1;
        const int n = (int)(dyn ? n4 : n3);
        if (n == 0) continue;
        const int64_t off = dyn ? n3 : 0;
        densify_apply_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
            dyn ? ctx->p4.as<float>() : ctx->p3.as<float>(), dyn ? ctx->m4.as<float>() : ctx->m3.as<float>(),
            dyn ? ctx->v4.as<float>() : ctx->v3.as<float>(), dyn ? ctx->cap4 : ctx->cap3,
            dyn ? np4.as<float>() : np3.as<float>(), dyn ? nm4.as<float>() : nm3.as<float>(),
            dyn ? nv4.as<float>() : nv3.as<float>(), dyn ? cap4 : cap3, n, dyn ? 1 : 0, dyn ? r4 : r3,
            ctx->dens_cat.as<uint8_t>() + off, base + 4 * N + off, base + 3 * N + off, dyn ? jit4 : jit3,
            log_split);
        count_launch();
        CKL();
    }
    CK(cudaStreamSynchronize(st));
    std::swap(ctx->p4, np4);
    std::swap(ctx->m4, nm4);
    std::swap(ctx->v4, nv4);
    std::swap(ctx->p3, np3);
    std::swap(ctx->m3, nm3);
    std::swap(ctx->v3, nv3);
    for (DBuf* b : {&np4, &nm4, &nv4, &np3, &nm3, &nv3}) b->release();
    ctx->n4 = nn4;
    ctx->n3 = nn3;
    ctx->cap4 = cap4;
    ctx->cap3 = cap3;
    for (DBuf* b : {&ctx->p4_alt, &ctx->m4_alt, &ctx->v4_alt}) CK(b->ensure((size_t)r4 * cap4 * 4));
    hgs_status r = hgs_layout_state(ctx);  // gradients and statistics restart at zero (train.cpp:239-240, 296-297)
    if (r != HGS_OK) return r;
    CK(cudaStreamSynchronize(st));
    return HGS_OK;
}

hgs_status hgs_opacity_reset(hgs_ctx* ctx, double floor_logit) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    if (ctx->n3)
        opacity_cap_kernel<<<(unsigned)((ctx->n3 + 255) / 256), 256, 0, ctx->stream>>>(
            ctx->p3.as<float>(), ctx->cap3, R3_OP, (int)ctx->n3, (float)floor_logit);
    if (ctx->n4)
        opacity_cap_kernel<<<(unsigned)((ctx->n4 + 255) / 256), 256, 0, ctx->stream>>>(
            ctx->p4.as<float>(), ctx->cap4, R4_OP, (int)ctx->n4, (float)floor_logit);
    count_launch(2);
    CKL();
    CK(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

}  // extern "C"
