// capi.cu -- the C ABI (include/hgs_gpu.h): context, scene residency, and
// the render pipeline orchestration.  Host code here is compiled with
// -ffp-contract=off: the camera position and the conversion threshold it
// computes must round exactly like the oracle's.
#include <algorithm>
#include <cmath>
#include <vector>
#include <cstdio>
#include <cstring>
#include <string>

#include "ctx.cuh"
#include "kernels.cuh"
#include "primitives.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

hgs_status fail(hgs_ctx* ctx, hgs_status s, const std::string& m) {
    if (ctx) ctx->err = m;
    return s;
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            return fail(ctx, HGS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
    } while (0)

#define CKL()                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                    \
        if (e_ != cudaSuccess)                                                                  \
            return fail(ctx, HGS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

int64_t round_cap(int64_t n) { return ((n + 127) / 128) * 128 + 128; }

// ---------------------------------------------------------------- layout
struct FieldMap {
    size_t off;  // offsetof in hgs_host_scene
    int dim;     // components per Gaussian (-1 = 3K SH)
    int row;     // first SoA row
};
const FieldMap kDyn[] = {
    {offsetof(hgs_host_scene, mean_x), 3, R4_MEAN}, {offsetof(hgs_host_scene, mean_t), 1, R4_MT},
    {offsetof(hgs_host_scene, ql), 4, R4_QL},       {offsetof(hgs_host_scene, qr), 4, R4_QR},
    {offsetof(hgs_host_scene, log_s4), 4, R4_LS},   {offsetof(hgs_host_scene, op4), 1, R4_OP},
    {offsetof(hgs_host_scene, sh4), -1, R4_SH},
};
const FieldMap kSta[] = {
    {offsetof(hgs_host_scene, mean3), 3, R3_MEAN}, {offsetof(hgs_host_scene, quat3), 4, R3_Q},
    {offsetof(hgs_host_scene, log_s3), 3, R3_LS},  {offsetof(hgs_host_scene, op3), 1, R3_OP},
    {offsetof(hgs_host_scene, sh3), -1, R3_SH},
};

void* field_ptr(const hgs_host_scene* s, const FieldMap& f) {
    return *reinterpret_cast<void* const*>(reinterpret_cast<const char*>(s) + f.off);
}

template <typename T>
__global__ void aos_to_soa_kernel(const T* __restrict__ src, int64_t n, int d, float* __restrict__ dst, int64_t cap,
                                  int row0) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t i = e / d;
    const int k = (int)(e - i * d);
    dst[(int64_t)(row0 + k) * cap + i] = (float)src[e];
}

template <typename T>
__global__ void soa_to_aos_kernel(const float* __restrict__ src, int64_t n, int d, int64_t cap, int row0,
                                  T* __restrict__ dst) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * d) return;
    const int64_t i = e / d;
    const int k = (int)(e - i * d);
    dst[e] = (T)src[(int64_t)(row0 + k) * cap + i];
}

// Host -> device SoA rows for one pool.
hgs_status upload_pool(hgs_ctx* ctx, const hgs_host_scene* s, const FieldMap* fm, int nf, int64_t n, int64_t cap,
                       float* dst, int dtype) {
    const int K3 = 3 * sh_count(ctx->deg);
    const size_t esz = dtype == HGS_F64 ? 8 : 4;
    for (int f = 0; f < nf; ++f) {
        const int d = fm[f].dim < 0 ? K3 : fm[f].dim;
        const void* src = field_ptr(s, fm[f]);
        if (n == 0) continue;
        if (!src) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "scene upload: null field pointer");
        const size_t bytes = (size_t)n * d * esz;
        CK(ctx->stage.ensure(bytes));
        CK(cudaMemcpyAsync(ctx->stage.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
        const int64_t tot = n * d;
        const int blocks = (int)((tot + 255) / 256);
        if (dtype == HGS_F64)
            aos_to_soa_kernel<double><<<blocks, 256, 0, ctx->stream>>>(ctx->stage.as<double>(), n, d, dst, cap,
                                                                      fm[f].row);
        else
            aos_to_soa_kernel<float><<<blocks, 256, 0, ctx->stream>>>(ctx->stage.as<float>(), n, d, dst, cap,
                                                                     fm[f].row);
        count_launch();
        CKL();
    }
    return HGS_OK;
}

hgs_status download_pool(hgs_ctx* ctx, hgs_host_scene* s, const FieldMap* fm, int nf, int64_t n, int64_t cap,
                         const float* src, int dtype) {
    const int K3 = 3 * sh_count(ctx->deg);
    const size_t esz = dtype == HGS_F64 ? 8 : 4;
    for (int f = 0; f < nf; ++f) {
        const int d = fm[f].dim < 0 ? K3 : fm[f].dim;
        void* dst = field_ptr(s, fm[f]);
        if (n == 0 || !dst) continue;
        const size_t bytes = (size_t)n * d * esz;
        CK(ctx->stage.ensure(bytes));
        const int64_t tot = n * d;
        const int blocks = (int)((tot + 255) / 256);
        if (dtype == HGS_F64)
            soa_to_aos_kernel<double><<<blocks, 256, 0, ctx->stream>>>(src, n, d, cap, fm[f].row,
                                                                      ctx->stage.as<double>());
        else
            soa_to_aos_kernel<float><<<blocks, 256, 0, ctx->stream>>>(src, n, d, cap, fm[f].row,
                                                                     ctx->stage.as<float>());
        count_launch();
        CKL();
        CK(cudaMemcpyAsync(dst, ctx->stage.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return HGS_OK;
}

// camera.hpp:21-26 Camera::validate
bool camera_valid(const hgs_camera* c, std::string& why) {
    if (!(c->fx > 0.0 && c->fy > 0.0)) return why = "Camera: fx, fy must be positive", false;
    if (!(0.0 < c->near_ && c->near_ < c->far_)) return why = "Camera: need 0 < near < far", false;
    if (c->width <= 0 || c->height <= 0) return why = "Camera: bad image dimensions", false;
    if (c->width > 32767 || c->height > 32767) return why = "Camera: image dimensions above 32767", false;
    const double* R = c->rot;
    double worst = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double s = R[0 * 3 + i] * R[0 * 3 + j];
            s = s + R[1 * 3 + i] * R[1 * 3 + j];
            s = s + R[2 * 3 + i] * R[2 * 3 + j];
            worst = std::fmax(worst, std::fabs(s - (i == j ? 1.0 : 0.0)));
        }
    const double det = R[0] * (R[4] * R[8] - R[5] * R[7]) - R[1] * (R[3] * R[8] - R[5] * R[6]) +
                       R[2] * (R[3] * R[7] - R[4] * R[6]);
    if (!(worst <= 1e-8 && std::fabs(det - 1.0) <= 1e-8)) return why = "Camera: rotation not orthonormal", false;
    return true;
}

DevCamera to_dev(const hgs_camera* c) {
    DevCamera d;
    d.fx = c->fx;
    d.fy = c->fy;
    d.cx = c->cx;
    d.cy = c->cy;
    for (int i = 0; i < 9; ++i) d.R[i] = c->rot[i];
    for (int i = 0; i < 3; ++i) d.t[i] = c->trans[i];
    for (int i = 0; i < 3; ++i) {  // camera.hpp:19 position() = -R^T t
        double s = (-c->rot[0 * 3 + i]) * c->trans[0];
        s = s + (-c->rot[1 * 3 + i]) * c->trans[1];
        s = s + (-c->rot[2 * 3 + i]) * c->trans[2];
        d.pos[i] = s;
    }
    d.width = c->width;
    d.height = c->height;
    d.near_ = c->near_;
    d.far_ = c->far_;
    return d;
}

__global__ void __launch_bounds__(256) zero_jobs_kernel(ZeroJobs J) {
    pdl_wait();  // launched with launch_pdl
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < J.n; ++k) {
        uint32_t* p = static_cast<uint32_t*>(J.j[k].p);
        const uint64_t n = J.j[k].words;
        const uint32_t v = J.j[k].value;
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = v;
    }
}

hgs_status check_flags(hgs_ctx* ctx, uint32_t flags) {
    if (flags & FLAG_NONUNIT_QUAT) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "quat_to_rot3: non-unit quaternion");
    if (flags & FLAG_INDEFINITE)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "clamp_psd: matrix is indefinite beyond rounding tolerance");
    if (flags & FLAG_NONUNIT_DIR) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "eval_sh: view direction must be unit");
    if (flags & FLAG_DEGENERATE_ROT)
        return fail(ctx, HGS_ERR_DEGENERATE_ROTATION, "extract_spatial_rot: spatial block is singular");
    if (flags & FLAG_NOT_ROTATION)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "rot3_to_quat: input is not a rotation matrix");
    return HGS_OK;
}

}  // namespace

// Row-major host rows -> given SoA destinations (used for Adam state upload).
hgs_status hgs_upload_rows(hgs_ctx* ctx, const hgs_host_scene* s, int dtype, float* dst4, float* dst3) {
    hgs_status r = upload_pool(ctx, s, kDyn, 7, ctx->n4, ctx->cap4, dst4, dtype);
    if (r != HGS_OK) return r;
    r = upload_pool(ctx, s, kSta, 5, ctx->n3, ctx->cap3, dst3, dtype);
    if (r != HGS_OK) return r;
    CK(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

// ---------------------------------------------------------------- profiler
void prof_begin(hgs_ctx* ctx, int phase) {
    if (!ctx->profile) return;
    cudaEvent_t a;
    if (ctx->ev_pool.empty()) cudaEventCreate(&a);
    else {
        a = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
    }
    cudaEventRecord(a, ctx->stream);
    ctx->ev_pending.push_back({phase, a, nullptr});
}

void prof_end(hgs_ctx* ctx) {
    if (!ctx->profile || ctx->ev_pending.empty() || ctx->ev_pending.back().b) return;
    cudaEvent_t b;
    if (ctx->ev_pool.empty()) cudaEventCreate(&b);
    else {
        b = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
    }
    cudaEventRecord(b, ctx->stream);
    ctx->ev_pending.back().b = b;
}

void prof_collect(hgs_ctx* ctx) {
    for (auto& e : ctx->ev_pending) {
        if (e.b) {
            cudaEventSynchronize(e.b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e.a, e.b);
            ctx->phase_ms[e.phase] += ms;
            ctx->phase_calls[e.phase] += 1;
            ctx->ev_pool.push_back(e.b);
        }
        ctx->ev_pool.push_back(e.a);
    }
    ctx->ev_pending.clear();
}

// ====================================================================== render
// The full K1 -> sort -> K2 -> sort -> K4 pipeline; leaves the tape in ctx.
namespace hgs {
#ifdef HGS_CHECKED
__device__ CheckCaps g_chk;
__device__ unsigned long long g_pairs[8];
void set_check_caps(const CheckCaps& caps, cudaStream_t st) {
    cudaMemcpyToSymbolAsync(g_chk, &caps, sizeof(CheckCaps), 0, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);  // (checked builds only) caps is a host temporary
}
#else
void set_check_caps(const CheckCaps&, cudaStream_t) {}
#endif
}  // namespace hgs

#ifdef HGS_CHECKED
namespace {
// Capacities (elements) of the render workspace for the checked build.
CheckCaps render_caps(const hgs_ctx* ctx, size_t npx, int n_tiles) {
    CheckCaps c;
    c.splats = std::min(ctx->rec_sorted.cap / sizeof(SplatRec), ctx->fast_sorted.cap / sizeof(SplatFast));
    if (ctx->accum.cap) c.splats = std::min<unsigned long long>(c.splats, ctx->accum.cap / (kAccStrideHost * sizeof(acc_t)));
    c.inst = std::min(std::min(ctx->inst_k.cap, ctx->inst_v.cap), std::min(ctx->inst_k2.cap, ctx->inst_v2.cap)) / 4;
    c.pixels = npx;
    c.tiles = (unsigned long long)n_tiles;
    return c;
}
}  // namespace
#endif

hgs_status hgs_render_pipeline(hgs_ctx* ctx, const hgs_camera* cam, double t, const double bg[3],
                               const hgs_raster_opts* opts, int deferred, uint32_t icap, void* counters_slot,
                               const ZeroJobs* extra) {
    std::string why;
    if (!camera_valid(cam, why)) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, why);
    const double cutoff = opts ? opts->weight_cutoff : 0.05;
    const bool want_count = opts && opts->count_map;
    const bool want_trans = opts && opts->transmittance_map;
    cudaStream_t st = ctx->stream;
    ctx->have_tape = false;
    ctx->stats_pending = false;
    const int n4 = (int)ctx->n4, n3 = (int)ctx->n3, N = n4 + n3;
    const int W = cam->width, H = cam->height;
    const int tiles_x = (W + kTile - 1) / kTile, tiles_y = (H + kTile - 1) / kTile;
    const int n_tiles = tiles_x * tiles_y;
    ctx->W = W;
    ctx->H = H;
    ctx->tiles_x = tiles_x;
    ctx->tiles_y = tiles_y;
    ctx->cam = to_dev(cam);
    ctx->t = t;
    for (int c = 0; c < 3; ++c) ctx->bg[c] = bg[c];

    const size_t npx = (size_t)W * H;
    CK(ctx->counters.ensure(sizeof(Counters)));
    CK(ctx->pinned_ctr.ensure(sizeof(Counters) + 64));
    Counters* dc = counters_slot ? static_cast<Counters*>(counters_slot) : ctx->counters.as<Counters>();
    Counters* hc = static_cast<Counters*>(ctx->pinned_ctr.p);
    ZeroJobs zj;
    if (extra) zj = *extra;
    zj.add(dc, sizeof(Counters));
    // capacity mode (icap > 0): no host round trip -- the duplication runs on
    // buffers for icap instances and flags FLAG_CAPACITY if that was too few
    // (the caller re-renders); only the production (culled) path supports it
    if (want_count || ctx->debug_full_list) icap = 0;
    CK(ctx->img.ensure(npx * 3 * sizeof(float)));
    CK(ctx->last.ensure(npx * sizeof(uint32_t)));
    CK(ctx->tfinal.ensure(npx * sizeof(float)));
    CK(ctx->fix_list.ensure(npx * sizeof(uint32_t)));
    CK(ctx->fix_cout.ensure(npx * 3 * sizeof(double)));
    CK(ctx->fix_slot.ensure(npx * sizeof(uint32_t)));
    if (want_trans) CK(ctx->trans.ensure(npx * sizeof(float)));
    if (want_count) CK(ctx->count.ensure(npx * sizeof(uint32_t)));
    CK(ctx->ranges.ensure((size_t)n_tiles * sizeof(uint2)));
    CK(ctx->tile_order.ensure((size_t)n_tiles * sizeof(uint32_t)));
    zj.add(ctx->ranges.p, (size_t)n_tiles * sizeof(uint2));
    if (N > 0 && !ctx->skip_gid_map) {  // (the backward's gid -> sorted index map)
        CK(ctx->sorted_of_gid.ensure((size_t)N * 4));
        zj.add(ctx->sorted_of_gid.p, (size_t)N * 4, 0xffffffffu);  // gather writes the visible ones
    }
    {
        uint64_t words = 0;
        for (int k = 0; k < zj.n; ++k) words += zj.j[k].words;
        const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((words + 255) / 256, ctx->sms * 8));
        CK(launch_pdl(zero_jobs_kernel, dim3(blocks), dim3(256), 0, st, zj));
        count_launch();
    }

    int64_t V = 0, I = 0;
    if (N > 0) {
        CK(ctx->rec.ensure((size_t)N * sizeof(SplatRec)));
        CK(ctx->depth_key.ensure((size_t)N * 4));
        CK(ctx->ntiles.ensure((size_t)N * 4));
        CK(ctx->visflag.ensure((size_t)N * 4));
        CK(ctx->vispos.ensure((size_t)N * 4));
        CK(ctx->shdir.ensure((size_t)N * sizeof(ShRec)));
        CK(ctx->scan_ws.ensure(scan_workspace_bytes(N) + 4096));
        prof_begin(ctx, PH_PREPROCESS);
        CK(preprocess_setup());
        CK(launch_pdl(ctx->skip_gid_map ? preprocess_render_kernel : preprocess_kernel, dim3(div_up(N, 256)),
                      dim3(256), preprocess_smem_bytes(ctx->deg), st,
                      static_cast<const float*>(ctx->p4.as<float>()), ctx->cap4, n4,
                      static_cast<const float*>(ctx->p3.as<float>()), ctx->cap3, n3, ctx->deg, ctx->cam, t, cutoff,
                      tiles_x, ctx->rec.as<SplatRec>(), ctx->depth_key.as<uint32_t>(), ctx->ntiles.as<uint32_t>(),
                      dc->stats, &dc->flags, ctx->shdir.as<ShRec>()));
        count_launch();
        CKL();
        // the visible count V stays on the device: buffers are sized for N,
        // the sort, gather and offset scan read V from device memory
        CK(ctx->sort_k.ensure((size_t)N * 4));
        CK(ctx->sort_v.ensure((size_t)N * 4));
        CK(ctx->sort_k2.ensure((size_t)N * 4));
        CK(ctx->sort_v2.ensure((size_t)N * 4));
        // the visible Gaussians' (depth key, index) in index order, V
        compact_visible(ctx->ntiles.as<uint32_t>(), ctx->depth_key.as<uint32_t>(), N, ctx->sort_k.as<uint32_t>(),
                        ctx->sort_v.as<uint32_t>(), &dc->V, ctx->scan_ws.as<uint32_t>(), st);
        CKL();
        prof_end(ctx);
        prof_begin(ctx, PH_DEPTH_SORT);
        CK(ctx->sort_ws.ensure(radix_workspace_bytes(N) + 4096));
        // stable sort by f32 depth bits; gid (projected order) breaks ties
        int which = radix_sort_pairs(ctx->sort_k.as<uint32_t>(), ctx->sort_v.as<uint32_t>(), ctx->sort_k2.as<uint32_t>(),
                                     ctx->sort_v2.as<uint32_t>(), N, 0, 32, ctx->sort_ws.as<uint32_t>(), st, &dc->V);
        CKL();
        prof_end(ctx);
        uint32_t* sorted_gid = which ? ctx->sort_v2.as<uint32_t>() : ctx->sort_v.as<uint32_t>();
        ctx->sorted_gid = sorted_gid;
        CK(ctx->rec_sorted.ensure((size_t)N * sizeof(SplatRec)));
        CK(ctx->fast_sorted.ensure((size_t)N * sizeof(SplatFast)));
        CK(ctx->ntiles_sorted.ensure((size_t)N * 4));
        CK(ctx->inst_off.ensure((size_t)N * 4));
        CK(ctx->sorted_of_gid.ensure((size_t)N * 4));
        CK(ctx->pcut.ensure((size_t)N * sizeof(CullRec)));
        prof_begin(ctx, PH_DUPLICATE);
        CK(launch_pdl(gather_sorted_kernel, dim3(div_up((uint32_t)N, 256)), dim3(256), 0, st,
            sorted_gid, &dc->V, ctx->rec.as<SplatRec>(), ctx->ntiles.as<uint32_t>(),
            ctx->skip_gid_map ? nullptr : ctx->rec_sorted.as<SplatRec>(),
            ctx->fast_sorted.as<SplatFast>(), ctx->ntiles_sorted.as<uint32_t>(), ctx->skip_gid_map ? nullptr : ctx->sorted_of_gid.as<uint32_t>(),
            ctx->pcut.as<CullRec>()));
        count_launch();
        CKL();
        exclusive_scan_u32(ctx->ntiles_sorted.as<uint32_t>(), ctx->inst_off.as<uint32_t>(), N, &dc->I,
                           ctx->scan_ws.as<uint32_t>(), st, &dc->V);
        CKL();
        prof_end(ctx);
        if (icap) {
            V = N;  // bounds only; the kernels read the true counts on the device
            I = icap;
        } else {
            // the one host round trip of a render: the instance count sizes the
            // duplication buffers; the preprocess error flags are reported here,
            // before anything downstream runs (the reference throws in K1)
            CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            V = hc->V;
            I = V ? hc->I : 0;
            hgs_status fs = check_flags(ctx, hc->flags);
            if (fs != HGS_OK) return fs;
        }
    }
    ctx->V = V;
    ctx->I = I;
    uint32_t* inst_vals = nullptr;
    if (I > 0) {
        CK(ctx->inst_k.ensure((size_t)I * 4));
        CK(ctx->inst_v.ensure((size_t)I * 4));
        CK(ctx->inst_k2.ensure((size_t)I * 4));
        CK(ctx->inst_v2.ensure((size_t)I * 4));
#ifdef HGS_CHECKED
        set_check_caps(render_caps(ctx, npx, n_tiles), st);
#endif
        const int cull = want_count ? 0 : 1;  // count_map counts every box-covered splat
        const uint32_t dup_blocks = div_up((uint32_t)I, kDupPerCtaHost);
        CK(ctx->dup_first.ensure((size_t)(dup_blocks + 1) * 4));
        if (cull && !ctx->debug_full_list) {
            // production path: duplication + exact culling + order-preserving
            // compaction in one kernel, then the stable tile sort of the kept
            prof_begin(ctx, PH_DUPLICATE);
            CK(ctx->dup_status.ensure((size_t)dup_blocks * 8 + 64));
            unsigned long long* status = ctx->dup_status.as<unsigned long long>();
            uint32_t* counter = reinterpret_cast<uint32_t*>(status + dup_blocks);
            CK(launch_pdl(dup_bounds_kernel, dim3(div_up((uint32_t)V, 256)), dim3(256), 0, st,
                          static_cast<const uint32_t*>(ctx->inst_off.as<uint32_t>()),
                          static_cast<const uint32_t*>(ctx->ntiles_sorted.as<uint32_t>()), (int)V,
                          ctx->dup_first.as<uint32_t>(), static_cast<const uint32_t*>(icap ? &dc->V : nullptr),
                          dup_blocks, reinterpret_cast<uint32_t*>(status), dup_blocks * 2 + 1));
            count_launch();
            CK(launch_pdl(duplicate_compact_kernel, dim3(dup_blocks), dim3(256), 0, st, ctx->fast_sorted.as<SplatFast>(),
                          (int)V, ctx->inst_off.as<uint32_t>(), tiles_x, ctx->pcut.as<CullRec>(),
                          ctx->dup_first.as<uint32_t>(), (int)I, ctx->inst_k2.as<uint32_t>(), ctx->inst_v2.as<uint32_t>(),
                          &dc->I_kept, status, counter, icap ? &dc->V : nullptr, icap ? &dc->I : nullptr,
                          &dc->flags));
            count_launch();
            CKL();
            prof_end(ctx);
            prof_begin(ctx, PH_TILE_SORT);
            int bits = 1;
            while ((1 << bits) < n_tiles) ++bits;
            const int end_bit = ((bits + 7) / 8) * 8;
            CK(ctx->sort_ws.ensure(radix_workspace_bytes((int)I) + 4096));
            ctx->inst_keys_all = ctx->inst_vals_all = nullptr;
            // the sort's last phase also writes the tile ranges
            int which = radix_sort_pairs(ctx->inst_k2.as<uint32_t>(), ctx->inst_v2.as<uint32_t>(),
                                         ctx->inst_k.as<uint32_t>(), ctx->inst_v.as<uint32_t>(), (int)I, 0, end_bit,
                                         ctx->sort_ws.as<uint32_t>(), st, &dc->I_kept, ctx->ranges.as<uint2>());
            CKL();
            inst_vals = which ? ctx->inst_v.as<uint32_t>() : ctx->inst_v2.as<uint32_t>();
            prof_end(ctx);
        } else {
        prof_begin(ctx, PH_DUPLICATE);
        if (cull) {
            CK(ctx->inst_flag.ensure((size_t)I * 4));
            CK(ctx->inst_pos.ensure((size_t)I * 4));
        }
        dup_bounds_kernel<<<div_up((uint32_t)V, 256), 256, 0, st>>>(
            ctx->inst_off.as<uint32_t>(), ctx->ntiles_sorted.as<uint32_t>(), (int)V, ctx->dup_first.as<uint32_t>(),
            nullptr, dup_blocks, nullptr, 0u);
        count_launch();
        duplicate_kernel<<<dup_blocks, 256, 0, st>>>(
            ctx->fast_sorted.as<SplatFast>(), ctx->rec_sorted.as<SplatRec>(), (int)V, ctx->inst_off.as<uint32_t>(),
            tiles_x, cull, ctx->pcut.as<CullRec>(), ctx->inst_k.as<uint32_t>(), ctx->inst_v.as<uint32_t>(),
            cull ? ctx->inst_flag.as<uint32_t>() : nullptr, ctx->dup_first.as<uint32_t>(), (int)I);
        count_launch();
        CKL();
        prof_end(ctx);
        prof_begin(ctx, PH_TILE_SORT);
        int bits = 1;
        while ((1 << bits) < n_tiles) ++bits;
        const int end_bit = ((bits + 7) / 8) * 8;
        CK(ctx->sort_ws.ensure(radix_workspace_bytes((int)I) + 4096));
        ctx->inst_keys_all = ctx->inst_vals_all = nullptr;
        if (ctx->debug_full_list || !cull) {
            // the reference's complete instance list (raster.cpp:180-212): kept for
            // count_map and for the bit-exact parity check (hgs_debug_instances)
            CK(ctx->dbg_k.ensure((size_t)I * 4));
            CK(ctx->dbg_v.ensure((size_t)I * 4));
            CK(cudaMemcpyAsync(ctx->dbg_k.p, ctx->inst_k.p, (size_t)I * 4, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(ctx->dbg_v.p, ctx->inst_v.p, (size_t)I * 4, cudaMemcpyDeviceToDevice, st));
            int w = radix_sort_pairs(ctx->dbg_k.as<uint32_t>(), ctx->dbg_v.as<uint32_t>(), ctx->inst_k2.as<uint32_t>(),
                                     ctx->inst_v2.as<uint32_t>(), (int)I, 0, end_bit, ctx->sort_ws.as<uint32_t>(), st);
            CKL();
            if (w) {
                CK(cudaMemcpyAsync(ctx->dbg_k.p, ctx->inst_k2.p, (size_t)I * 4, cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(ctx->dbg_v.p, ctx->inst_v2.p, (size_t)I * 4, cudaMemcpyDeviceToDevice, st));
            }
            ctx->inst_keys_all = ctx->dbg_k.as<uint32_t>();
            ctx->inst_vals_all = ctx->dbg_v.as<uint32_t>();
        }
        uint32_t* keys;
        if (cull) {
            // Exact culling first (order-preserving compaction of the depth-ordered
            // instances that can reach the alpha cutoff in their tile), then the
            // stable tile sort of the kept instances only: same relative order as
            // filtering the reference's sorted list, at a third of the sort cost.
            CK(ctx->scan_ws.ensure(scan_workspace_bytes((int)I) + 4096));
            exclusive_scan_u32(ctx->inst_flag.as<uint32_t>(), ctx->inst_pos.as<uint32_t>(), (int)I, &dc->I_kept,
                               ctx->scan_ws.as<uint32_t>(), st);
            compact_instances_kernel<<<div_up((uint32_t)I, 256), 256, 0, st>>>(
                ctx->inst_k.as<uint32_t>(), ctx->inst_v.as<uint32_t>(), (int)I, ctx->inst_pos.as<uint32_t>(),
                ctx->inst_k2.as<uint32_t>(), ctx->inst_v2.as<uint32_t>());
            count_launch();
            CKL();
            int which = radix_sort_pairs(ctx->inst_k2.as<uint32_t>(), ctx->inst_v2.as<uint32_t>(),
                                         ctx->inst_k.as<uint32_t>(), ctx->inst_v.as<uint32_t>(), (int)I, 0, end_bit,
                                         ctx->sort_ws.as<uint32_t>(), st, &dc->I_kept);
            CKL();
            keys = which ? ctx->inst_k.as<uint32_t>() : ctx->inst_k2.as<uint32_t>();
            inst_vals = which ? ctx->inst_v.as<uint32_t>() : ctx->inst_v2.as<uint32_t>();
            CK(launch_pdl(tile_ranges_dev_kernel, dim3(div_up((uint32_t)I, 256)), dim3(256), 0, st,
                          static_cast<const uint32_t*>(keys), static_cast<const uint32_t*>(&dc->I_kept),
                          ctx->ranges.as<uint2>()));
            count_launch();
        } else {
            keys = ctx->inst_keys_all;
            inst_vals = ctx->inst_vals_all;
            tile_ranges_kernel<<<div_up((uint32_t)I, 256), 256, 0, st>>>(keys, (int)I, ctx->ranges.as<uint2>());
            count_launch();
        }
        CKL();
        prof_end(ctx);
        }
    }
    ctx->inst_vals_final = inst_vals;
#ifdef HGS_CHECKED
    set_check_caps(render_caps(ctx, npx, n_tiles), st);
#endif
    prof_begin(ctx, PH_RASTER_FWD);
    launch_raster_fwd(
        want_count, n_tiles, st, ctx->ranges.as<uint2>(), inst_vals, ctx->fast_sorted.as<SplatFast>(),
        ctx->skip_gid_map ? ctx->rec.as<SplatRec>() : ctx->rec_sorted.as<SplatRec>(), W, H,
        tiles_x, (float)bg[0], (float)bg[1], (float)bg[2], ctx->img.as<float>(), ctx->last.as<uint32_t>(),
        ctx->tfinal.as<float>(), want_trans ? ctx->trans.as<float>() : nullptr, want_count ? ctx->count.as<uint32_t>() : nullptr,
        ctx->fix_list.as<uint32_t>(), &dc->fix_count, tile_order_enabled() ? ctx->tile_order.as<uint32_t>() : nullptr,
        bg[0], bg[1], bg[2], ctx->fix_cout.as<double>(), ctx->fix_slot.as<uint32_t>(),
        ctx->skip_gid_map ? ctx->sorted_gid : nullptr);
    count_launch();
    CKL();
    prof_end(ctx);
    ctx->have_tape = true;
    ctx->stats_pending = true;
    if (deferred) return HGS_OK;
    return hgs_render_finish(ctx);
}

// Reads the counters of the last render (RenderStats, fix-up and kept
// counts, error flags): one stream synchronisation, skipped by the training
// step until its end.
hgs_status hgs_render_finish(hgs_ctx* ctx) {
    if (!ctx->stats_pending) return HGS_OK;
    ctx->stats_pending = false;
    Counters* dc = ctx->counters.as<Counters>();
    Counters* hc = static_cast<Counters*>(ctx->pinned_ctr.p);
    CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->stats.culled_depth = (int64_t)hc->stat(0);
    ctx->stats.culled_offscreen = (int64_t)hc->stat(1);
    ctx->stats.culled_degenerate = (int64_t)hc->stat(2);
    ctx->stats.culled_temporal = (int64_t)hc->stat(3);
    ctx->stats.degenerate_temporal = (int64_t)hc->stat(4);
    ctx->stats.projected = (int64_t)hc->stat(5);
    ctx->fixups = hc->fix_count;
    ctx->kept = ctx->I ? (int64_t)hc->I_kept : 0;
    hgs_status s = check_flags(ctx, hc->flags);
    if (s != HGS_OK) {
        ctx->have_tape = false;
        return s;
    }
    return HGS_OK;
}

// (Re)lays out the packed gradient buffer and the per-Gaussian statistics
// for the current capacities, all zero (upload, densification).
hgs_status hgs_layout_state(hgs_ctx* ctx) {
    {
        const int64_t f4 = (int64_t)rows4(ctx->deg) * ctx->cap4, f3 = (int64_t)rows3(ctx->deg) * ctx->cap3;
        ctx->gbuf_floats = f4 + f3 + 2 * ctx->cap4 + 2 * ctx->cap3;
        CK(ctx->gbuf.ensure((size_t)ctx->gbuf_floats * 4));
        CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
        ctx->grads_zero = true;
        float* g = ctx->gbuf.as<float>();
        ctx->g4 = g;
        ctx->g3 = g + f4;
        ctx->dgn4 = ctx->g3 + f3;
        ctx->dgn3 = ctx->dgn4 + ctx->cap4;
        ctx->dcnt4 = ctx->dgn3 + ctx->cap3;
        ctx->dcnt3 = ctx->dcnt4 + ctx->cap4;
    }
    for (DBuf* b : {&ctx->gn4, &ctx->cnt4, &ctx->sn4}) {
        CK(b->ensure((size_t)ctx->cap4 * 4));
        CK(cudaMemsetAsync(b->p, 0, (size_t)ctx->cap4 * 4, ctx->stream));
    }
    for (DBuf* b : {&ctx->gn3, &ctx->cnt3, &ctx->sn3}) {
        CK(b->ensure((size_t)ctx->cap3 * 4));
        CK(cudaMemsetAsync(b->p, 0, (size_t)ctx->cap3 * 4, ctx->stream));
    }
    ctx->have_tape = false;
    return HGS_OK;
}

extern "C" {

hgs_status hgs_profile(hgs_ctx* ctx, int enable) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    prof_collect(ctx);
    ctx->profile = enable != 0;
    return HGS_OK;
}

hgs_status hgs_profile_read(hgs_ctx* ctx, double* ms16, long long* calls16, int reset) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    for (int i = 0; i < 16; ++i) {
        if (ms16) ms16[i] = ctx->phase_ms[i];
        if (calls16) calls16[i] = ctx->phase_calls[i];
        if (reset) {
            ctx->phase_ms[i] = 0.0;
            ctx->phase_calls[i] = 0;
        }
    }
    return HGS_OK;
}

long long hgs_launch_count(void) { return launch_count(); }

hgs_status hgs_ctx_create(int device, hgs_ctx** out) {
    if (!out) return HGS_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        return HGS_ERR_CUDA;
    }
    if (device < 0 || device >= n) return HGS_ERR_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return HGS_ERR_CUDA;
    hgs_ctx* ctx = new hgs_ctx();
    ctx->device = device;
    if (const char* dbg = getenv("HGS_DEBUG_EXACT")) set_debug_exact(atoi(dbg));  // diagnostics only
    if (const char* dbg = getenv("HGS_DEBUG_TERR")) set_debug_terr((float)atof(dbg));
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return HGS_ERR_CUDA;
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return HGS_OK;
}

void hgs_ctx_destroy(hgs_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    hgs_comm_destroy(ctx);
    DBuf* bufs[] = {&ctx->p4, &ctx->p3, &ctx->p4_alt, &ctx->m4_alt, &ctx->v4_alt, &ctx->gbuf, &ctx->scratch, &ctx->m4, &ctx->v4, &ctx->m3, &ctx->v3, &ctx->gn4,
                    &ctx->gn3, &ctx->cnt4, &ctx->cnt3, &ctx->sn4, &ctx->sn3, &ctx->rec, &ctx->depth_key,
                    &ctx->ntiles, &ctx->visflag, &ctx->vispos, &ctx->sort_k, &ctx->sort_v, &ctx->sort_k2,
                    &ctx->sort_v2, &ctx->rec_sorted, &ctx->fast_sorted, &ctx->ntiles_sorted, &ctx->inst_off,
                    &ctx->inst_k, &ctx->inst_v, &ctx->inst_k2, &ctx->inst_v2, &ctx->ranges, &ctx->sorted_of_gid, &ctx->inst_flag, &ctx->inst_pos, &ctx->dbg_k, &ctx->dbg_v, &ctx->scan_ws,
                    &ctx->sort_ws, &ctx->counters, &ctx->img, &ctx->last, &ctx->tfinal, &ctx->trans, &ctx->count,
                    &ctx->fix_list, &ctx->accum, &ctx->exact_col, &ctx->loss_img, &ctx->lgrad, &ctx->gt_stage, &ctx->loss_ws, &ctx->stage, &ctx->adam_ok, &ctx->pcut, &ctx->dup_first, &ctx->shdir, &ctx->ddir, &ctx->dup_status, &ctx->gpack, &ctx->dens_cat, &ctx->dens_u32, &ctx->dens_misc, &ctx->dens_kinds, &ctx->dens_jit, &ctx->dmap, &ctx->ckpt, &ctx->crc_tab, &ctx->comm_buf, &ctx->sweep_ctr};
    for (DBuf* b : bufs) b->release();
    ctx->pinned.release();
    ctx->pinned_ctr.release();
    ctx->pinned_pipe.release();
    ctx->ckpt_host.release();
    ctx->sweep_host.release();
    for (int k = 0; k < HGS_TRAIN_PIPELINE; ++k)
        if (ctx->pipe_ev[k]) cudaEventDestroy(ctx->pipe_ev[k]);
    for (int b = 0; b < 2; ++b) {
        ctx->gt_buf[b].release();
        ctx->gt_stage64[b].release();
        if (ctx->gt_ready[b]) cudaEventDestroy(ctx->gt_ready[b]);
        if (ctx->gt_free[b]) cudaEventDestroy(ctx->gt_free[b]);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* hgs_last_error(const hgs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

hgs_status hgs_ctx_set_stream(hgs_ctx* ctx, void* stream) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return HGS_OK;
}

void* hgs_ctx_stream(hgs_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

hgs_status hgs_synchronize(hgs_ctx* ctx) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

}  // extern "C"

hgs_status hgs_scene_alloc(hgs_ctx* ctx, int64_t n4, int64_t n3, int deg, double tau, double extent,
                           double duration) {
    if (n4 < 0 || n3 < 0 || deg < 0 || deg > 3)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "scene upload: bad sizes or sh_degree (0..3)");
    if (n4 + n3 > (int64_t)INT32_MAX / 2) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "scene too large");
    ctx->state_sharded = false;  // fresh moments
    CK(cudaSetDevice(ctx->device));
    if (!ctx->pipeline.empty())
        return fail(ctx, HGS_ERR_STATE, "scene upload: collect the pipelined iterations first");
    ctx->n4 = n4;
    ctx->n3 = n3;
    ctx->deg = deg;
    ctx->tau = tau;
    ctx->extent = extent;
    ctx->duration = duration;
    ctx->cap4 = round_cap(n4);
    ctx->cap3 = round_cap(n3 + n4);  // room for every 4D Gaussian to convert
    const size_t b4 = (size_t)rows4(ctx->deg) * ctx->cap4 * sizeof(float);
    const size_t b3 = (size_t)rows3(ctx->deg) * ctx->cap3 * sizeof(float);
    for (DBuf* b : {&ctx->p4, &ctx->m4, &ctx->v4, &ctx->p4_alt, &ctx->m4_alt, &ctx->v4_alt}) CK(b->ensure(b4));
    for (DBuf* b : {&ctx->p3, &ctx->m3, &ctx->v3}) CK(b->ensure(b3));
    for (DBuf* b : {&ctx->m4, &ctx->v4}) CK(cudaMemsetAsync(b->p, 0, b4, ctx->stream));
    for (DBuf* b : {&ctx->m3, &ctx->v3}) CK(cudaMemsetAsync(b->p, 0, b3, ctx->stream));
    {
        hgs_status r = hgs_layout_state(ctx);
        if (r != HGS_OK) return r;
    }
    ctx->step = 0;
    ctx->have_tape = false;
    ctx->stats_pending = false;
    ctx->icap = 0;
    ctx->dens_planned = false;  // a densify plan belongs to the pools it was made for
    const uint64_t zero = 0;
    return hgs_skipped_total(ctx, nullptr, &zero);
}

extern "C" {

hgs_status hgs_scene_upload(hgs_ctx* ctx, const hgs_host_scene* s, int dtype) {
    if (!ctx || !s) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = hgs_scene_alloc(ctx, s->n4, s->n3, s->sh_degree, s->tau, s->extent, s->duration_seconds);
    if (r != HGS_OK) return r;
    r = upload_pool(ctx, s, kDyn, 7, ctx->n4, ctx->cap4, ctx->p4.as<float>(), dtype);
    if (r != HGS_OK) return r;
    r = upload_pool(ctx, s, kSta, 5, ctx->n3, ctx->cap3, ctx->p3.as<float>(), dtype);
    if (r != HGS_OK) return r;
    CK(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

hgs_status hgs_scene_download(hgs_ctx* ctx, hgs_host_scene* out, int dtype) {
    if (!ctx || !out) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = download_pool(ctx, out, kDyn, 7, ctx->n4, ctx->cap4, ctx->p4.as<float>(), dtype);
    if (r != HGS_OK) return r;
    r = download_pool(ctx, out, kSta, 5, ctx->n3, ctx->cap3, ctx->p3.as<float>(), dtype);
    if (r != HGS_OK) return r;
    out->n4 = ctx->n4;
    out->n3 = ctx->n3;
    out->sh_degree = ctx->deg;
    out->tau = ctx->tau;
    out->extent = ctx->extent;
    out->duration_seconds = ctx->duration;
    return HGS_OK;
}

// density_map (raster.cpp:268-287): K1 projects the pools (statics skipped
// when dynamics_only), every projected splat adds +1 over its clamped box
// through a 2D difference array, row and column prefix sums finish it.
// Reuses the render buffers, so the last render's tape is released.
hgs_status hgs_density_map(hgs_ctx* ctx, const hgs_camera* cam, double t, int dynamics_only, double weight_cutoff,
                           uint32_t* counts_host) {
    if (!ctx || !cam || !counts_host) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    std::string why;
    if (!camera_valid(cam, why)) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, why);
    hgs_status r = hgs_render_finish(ctx);
    if (r != HGS_OK) return r;
    ctx->have_tape = false;
    cudaStream_t st = ctx->stream;
    const int n4 = (int)ctx->n4, n3 = dynamics_only ? 0 : (int)ctx->n3, N = n4 + n3;
    const int W = cam->width, H = cam->height;
    const int tiles_x = (W + kTile - 1) / kTile;
    const size_t npx = (size_t)W * H, ndiff = (size_t)(W + 1) * (H + 1);
    CK(ctx->counters.ensure(sizeof(Counters)));
    CK(ctx->pinned_ctr.ensure(sizeof(Counters) + 64));
    Counters* dc = ctx->counters.as<Counters>();
    Counters* hc = static_cast<Counters*>(ctx->pinned_ctr.p);
    CK(cudaMemsetAsync(dc, 0, sizeof(Counters), st));
    CK(ctx->dmap.ensure((ndiff + npx) * 4));
    int* diff = ctx->dmap.as<int>();
    uint32_t* out = reinterpret_cast<uint32_t*>(diff + ndiff);
    CK(cudaMemsetAsync(diff, 0, ndiff * 4, st));
    if (N > 0) {
        CK(ctx->rec.ensure((size_t)N * sizeof(SplatRec)));
        CK(ctx->depth_key.ensure((size_t)N * 4));
        CK(ctx->ntiles.ensure((size_t)N * 4));
        CK(ctx->shdir.ensure((size_t)N * sizeof(ShRec)));
        CK(preprocess_setup());
        preprocess_render_kernel<<<div_up(N, 256), 256, preprocess_smem_bytes(ctx->deg), st>>>(
            ctx->p4.as<float>(), ctx->cap4, n4, ctx->p3.as<float>(), ctx->cap3, n3, ctx->deg, to_dev(cam), t,
            weight_cutoff, tiles_x, ctx->rec.as<SplatRec>(), ctx->depth_key.as<uint32_t>(), ctx->ntiles.as<uint32_t>(),
            dc->stats, &dc->flags, ctx->shdir.as<ShRec>());
        count_launch();
        CKL();
        density_diff_kernel<<<div_up(N, 256), 256, 0, st>>>(ctx->ntiles.as<uint32_t>(), ctx->rec.as<SplatRec>(), N, W,
                                                           H, diff);
        count_launch();
        CKL();
    }
    density_rows_kernel<<<div_up(H + 1, 8), 256, 0, st>>>(diff, W, H);
    count_launch();
    CKL();
    density_cols_kernel<<<div_up(W, 256), 256, 0, st>>>(diff, W, H, out);
    count_launch();
    CKL();
    CK(cudaMemcpyAsync(counts_host, out, npx * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc, dc, sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return check_flags(ctx, hc->flags);
}

hgs_status hgs_scene_counts(hgs_ctx* ctx, int64_t* n4, int64_t* n3, int32_t* deg) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (n4) *n4 = ctx->n4;
    if (n3) *n3 = ctx->n3;
    if (deg) *deg = ctx->deg;
    return HGS_OK;
}

// Render sweep (config c5: one scene, many (camera, t) frames): every frame in
// capacity mode -- no host round trip inside the sweep, one synchronisation
// at its end.  The instance capacity is learned from a synchronous first
// frame (and kept on the context); a frame that overflowed it is redone
// synchronously at the end with the exact size, so the outputs are always
// those of hgs_render.
hgs_status hgs_render_sweep(hgs_ctx* ctx, int n, const hgs_camera* cams, const double* ts, const double bg[3],
                            const hgs_raster_opts* opts, float* out, int out_on_device, hgs_render_stats* stats) {
    if (!ctx || n < 0 || (n > 0 && (!cams || !ts)) || !bg) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = hgs_render_finish(ctx);
    if (r != HGS_OK) return r;
    if (n == 0) return HGS_OK;
    std::string why;
    for (int f = 0; f < n; ++f) {
        if (!camera_valid(&cams[f], why)) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, why);
        if (out && (cams[f].width != cams[0].width || cams[f].height != cams[0].height))
            return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "render_sweep: frames of one output differ in size");
    }
    cudaStream_t st = ctx->stream;
    const size_t npx = (size_t)cams[0].width * cams[0].height;
    CK(ctx->sweep_ctr.ensure((size_t)n * sizeof(Counters)));
    CK(ctx->sweep_host.ensure((size_t)n * sizeof(Counters)));
    Counters* slots = ctx->sweep_ctr.as<Counters>();
    Counters* hs = static_cast<Counters*>(ctx->sweep_host.p);
    auto emit = [&](int f) -> cudaError_t {
        if (!out) return cudaSuccess;
        return cudaMemcpyAsync(out + (size_t)f * npx * 3, ctx->img.p, npx * 3 * 4,
                               out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st);
    };
    int f0 = 0;
    if (ctx->icap == 0) {  // learn the capacity from a synchronous first frame
        ctx->skip_gid_map = n > 1;
        r = hgs_render_pipeline(ctx, &cams[0], ts[0], bg, opts, 1, 0, &slots[0]);
        ctx->skip_gid_map = false;
        if (r != HGS_OK) return r;
        ctx->icap = (uint32_t)std::min<int64_t>(INT32_MAX / 2, std::max<int64_t>(4096, ctx->I + ctx->I / 4 + 4096));
        CK(emit(0));
        f0 = 1;
    }
    for (int f = f0; f < n; ++f) {
        ctx->skip_gid_map = f + 1 < n;  // only the last frame's tape is kept
        r = hgs_render_pipeline(ctx, &cams[f], ts[f], bg, opts, 1, ctx->icap, &slots[f]);
        ctx->skip_gid_map = false;
        if (r != HGS_OK) return r;
        CK(emit(f));
    }
    CK(cudaMemcpyAsync(hs, slots, (size_t)n * sizeof(Counters), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    prof_collect(ctx);
    ctx->stats_pending = false;
    uint32_t need = 0;
    for (int f = 0; f < n; ++f)
        if (hs[f].flags & FLAG_CAPACITY) need = std::max(need, hs[f].I);
    if (need) {  // redo the overflowed frames exactly, keep the larger capacity
        ctx->icap = (uint32_t)std::min<int64_t>(INT32_MAX / 2, (int64_t)need + need / 4 + 4096);
        for (int f = 0; f < n; ++f) {
            if (!(hs[f].flags & FLAG_CAPACITY)) continue;
            ctx->skip_gid_map = f + 1 < n;
            r = hgs_render_pipeline(ctx, &cams[f], ts[f], bg, opts, 1, 0, &slots[f]);
            ctx->skip_gid_map = false;
            if (r != HGS_OK) return r;
            CK(emit(f));
            CK(cudaMemcpyAsync(&hs[f], &slots[f], sizeof(Counters), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ctx->redone_frames++;
        }
        // the context's tape is the last frame's: render it again if it was not redone
        if (!(hs[n - 1].flags & FLAG_CAPACITY) && n > 1) {
            r = hgs_render_pipeline(ctx, &cams[n - 1], ts[n - 1], bg, opts, 1, 0, &slots[n - 1]);
            if (r != HGS_OK) return r;
            CK(cudaMemcpyAsync(&hs[n - 1], &slots[n - 1], sizeof(Counters), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
    }
    for (int f = 0; f < n; ++f) {
        r = check_flags(ctx, hs[f].flags);
        if (r != HGS_OK) {
            ctx->have_tape = false;
            return r;
        }
        if (stats) {
            hgs_render_stats& o = stats[f];
            o.culled_depth = (int64_t)hs[f].stat(0);
            o.culled_offscreen = (int64_t)hs[f].stat(1);
            o.culled_degenerate = (int64_t)hs[f].stat(2);
            o.culled_temporal = (int64_t)hs[f].stat(3);
            o.degenerate_temporal = (int64_t)hs[f].stat(4);
            o.projected = (int64_t)hs[f].stat(5);
        }
    }
    const Counters& last = hs[n - 1];
    ctx->stats.culled_depth = (int64_t)last.stat(0);
    ctx->stats.culled_offscreen = (int64_t)last.stat(1);
    ctx->stats.culled_degenerate = (int64_t)last.stat(2);
    ctx->stats.culled_temporal = (int64_t)last.stat(3);
    ctx->stats.degenerate_temporal = (int64_t)last.stat(4);
    ctx->stats.projected = (int64_t)last.stat(5);
    ctx->fixups = last.fix_count;
    ctx->kept = last.I_kept;
    ctx->V = last.V;
    ctx->I = last.I;
    return HGS_OK;
}

hgs_status hgs_render(hgs_ctx* ctx, const hgs_camera* cam, double t, const double bg[3], const hgs_raster_opts* opts,
                      float* rgb_host, uint32_t* count_host, float* trans_host, hgs_render_stats* stats) {
    if (!ctx || !cam || !bg) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = hgs_render_pipeline(ctx, cam, t, bg, opts);
    if (r != HGS_OK) return r;
    const size_t npx = (size_t)ctx->W * ctx->H;
    if (rgb_host) CK(cudaMemcpyAsync(rgb_host, ctx->img.p, npx * 3 * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (count_host && opts && opts->count_map)
        CK(cudaMemcpyAsync(count_host, ctx->count.p, npx * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (trans_host && opts && opts->transmittance_map)
        CK(cudaMemcpyAsync(trans_host, ctx->trans.p, npx * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    prof_collect(ctx);
    if (stats) *stats = ctx->stats;
    return HGS_OK;
}

hgs_status hgs_rasterize(hgs_ctx* ctx, const hgs_host_scene* scene, int dtype, const hgs_camera* cam, double t,
                         const double bg[3], const hgs_raster_opts* opts, void* rgb_out, uint32_t* count_out,
                         void* trans_out, hgs_render_stats* stats) {
    if (!ctx || !scene || !cam || !bg) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = hgs_scene_upload(ctx, scene, dtype);
    if (r != HGS_OK) return r;
    const size_t npx = (size_t)cam->width * cam->height;
    std::vector<float> rgb(rgb_out ? npx * 3 : 0), trans(trans_out ? npx : 0);
    r = hgs_render(ctx, cam, t, bg, opts, rgb_out ? rgb.data() : nullptr, count_out,
                   trans_out ? trans.data() : nullptr, stats);
    if (r != HGS_OK) return r;
    if (rgb_out) {
        if (dtype == HGS_F64)
            for (size_t i = 0; i < rgb.size(); ++i) static_cast<double*>(rgb_out)[i] = rgb[i];
        else
            std::memcpy(rgb_out, rgb.data(), rgb.size() * 4);
    }
    if (trans_out) {
        if (dtype == HGS_F64)
            for (size_t i = 0; i < trans.size(); ++i) static_cast<double*>(trans_out)[i] = trans[i];
        else
            std::memcpy(trans_out, trans.data(), trans.size() * 4);
    }
    return HGS_OK;
}

const float* hgs_last_image_device(hgs_ctx* ctx) { return ctx ? ctx->img.as<float>() : nullptr; }

hgs_status hgs_set_exact_backward(hgs_ctx* ctx, int enable) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    ctx->exact_backward = enable != 0;
    return HGS_OK;
}

hgs_status hgs_render_info_get(hgs_ctx* ctx, hgs_render_info* info) {
    if (!ctx || !info) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = hgs_render_finish(ctx);
    if (r != HGS_OK) return r;
    info->visible = ctx->V;
    info->instances = ctx->I;
    info->fixup_pixels = ctx->fixups;
    info->kept_instances = ctx->kept;
    info->sweep_redone_frames = ctx->redone_frames;
    return HGS_OK;
}

// ---- parity introspection (used by tests/, not part of the reference API)
// Projected splats in projected-index order: gid, f32 depth bits, box, mean,
// conic, alpha, rgb.
hgs_status hgs_debug_splats(hgs_ctx* ctx, int32_t* gid, uint32_t* depth_bits, int32_t* box4, double* mean2,
                            double* conic4, double* alpha, float* rgb, int64_t cap, int64_t* n_out) {
    if (!ctx || !ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "no render to inspect");
    const int64_t V = ctx->V;
    *n_out = V;
    if (V > cap || V == 0) return HGS_OK;
    std::vector<uint32_t> sg(V);
    std::vector<SplatRec> rs(V);
    CK(cudaMemcpy(sg.data(), ctx->sorted_gid, V * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rs.data(), ctx->rec_sorted.p, V * sizeof(SplatRec), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> dk(ctx->n4 + ctx->n3);
    CK(cudaMemcpy(dk.data(), ctx->depth_key.p, dk.size() * 4, cudaMemcpyDeviceToHost));
    // projected order = increasing gid
    std::vector<int64_t> order(V);
    for (int64_t j = 0; j < V; ++j) order[j] = j;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sg[a] < sg[b]; });
    for (int64_t q = 0; q < V; ++q) {
        const int64_t j = order[q];
        const SplatRec& e = rs[j];
        gid[q] = (int32_t)sg[j];
        depth_bits[q] = dk[sg[j]];
        box4[q * 4 + 0] = e.x0;
        box4[q * 4 + 1] = e.x1;
        box4[q * 4 + 2] = e.y0;
        box4[q * 4 + 3] = e.y1;
        mean2[q * 2 + 0] = e.sx;
        mean2[q * 2 + 1] = e.sy;
        conic4[q * 4 + 0] = e.c00;
        conic4[q * 4 + 1] = e.c01;
        conic4[q * 4 + 2] = e.c10;
        conic4[q * 4 + 3] = e.c11;
        alpha[q] = e.alpha;
        rgb[q * 3 + 0] = e.r;
        rgb[q * 3 + 1] = e.g;
        rgb[q * 3 + 2] = e.b;
    }
    return HGS_OK;
}

// Keep the reference's complete tile-sorted instance list on subsequent
// renders (an extra sort of every instance; parity tests only).
// Test hook: the instance capacity the next hgs_render_sweep frames are
// launched with (0 = learn it from a synchronous first frame).
hgs_status hgs_debug_set_sweep_capacity(hgs_ctx* ctx, int64_t capacity) {
    if (!ctx || capacity < 0 || capacity > INT32_MAX / 2) return HGS_ERR_INVALID_ARGUMENT;
    ctx->icap = (uint32_t)capacity;
    return HGS_OK;
}

hgs_status hgs_debug_pair_counters(hgs_ctx* ctx, unsigned long long out[8], int reset) {
    if (!ctx || !out) return HGS_ERR_INVALID_ARGUMENT;
#ifdef HGS_CHECKED
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpyFromSymbol(out, g_pairs, 8 * sizeof(unsigned long long)));
    if (reset) {
        const unsigned long long z[8] = {};
        CK(cudaMemcpyToSymbol(g_pairs, z, sizeof(z)));
    }
    return HGS_OK;
#else
    return fail(ctx, HGS_ERR_STATE, "pair counters exist in the checked build only (libhgs_gpu_checked.so)");
#endif
}

hgs_status hgs_debug_keep_instances(hgs_ctx* ctx, int enable) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    ctx->debug_full_list = enable != 0;
    return HGS_OK;
}

// Tile-sorted instances: tile id and gid of each, in reference order.
hgs_status hgs_debug_instances(hgs_ctx* ctx, uint32_t* tile, uint32_t* gid, int64_t cap, int64_t* n_out) {
    if (!ctx || !ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "no render to inspect");
    const int64_t I = ctx->I, V = ctx->V;
    *n_out = I;
    if (I > cap || I == 0) return HGS_OK;
    if (!ctx->inst_vals_all)
        return fail(ctx, HGS_ERR_STATE, "full instance list not kept: call hgs_debug_keep_instances(ctx, 1) first");
    std::vector<uint32_t> vals(I), sg(V);
    CK(cudaMemcpy(vals.data(), ctx->inst_vals_all, I * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(sg.data(), ctx->sorted_gid, V * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tile, ctx->inst_keys_all, I * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < I; ++i) gid[i] = sg[vals[i] & hgs::kInstIndexMask];
    return HGS_OK;
}

// The 8x8-quadrant contribution mask of every instance of the full list
// (same order as hgs_debug_instances): bit q = quadrant (q & 1, q >> 1).
hgs_status hgs_debug_instance_masks(hgs_ctx* ctx, uint8_t* masks, int64_t cap, int64_t* n_out) {
    if (!ctx || !n_out || !ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "no render to inspect");
    const int64_t I = ctx->I;
    *n_out = I;
    if (I > cap || I == 0) return HGS_OK;
    if (!ctx->inst_vals_all)
        return fail(ctx, HGS_ERR_STATE, "full instance list not kept: call hgs_debug_keep_instances(ctx, 1) first");
    std::vector<uint32_t> vals(I);
    CK(cudaMemcpy(vals.data(), ctx->inst_vals_all, I * 4, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < I; ++i) masks[i] = (uint8_t)(vals[i] >> hgs::kInstMaskShift);
    return HGS_OK;
}

}  // extern "C"

namespace hgs {
// programmatic dependent launches (raster_common.cuh launch_pdl): on unless HGS_NO_PDL is set
bool tile_order_enabled() {  // HGS_NO_TILE_ORDER=1: row-major tile launch order
    static const bool on = !getenv("HGS_NO_TILE_ORDER");
    return on;
}

bool pdl_enabled() {
    static const bool on = getenv("HGS_NO_PDL") == nullptr;
    return on;
}
}  // namespace hgs
