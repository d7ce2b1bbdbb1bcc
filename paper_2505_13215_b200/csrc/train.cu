// train.cu -- training entry points of the C ABI: forward_train / backward
// (backward.hpp:68-74), loss (loss.hpp:12-13), Adam (train.hpp:68-69),
// conversion sweep (scene.hpp:75 + train.cpp:305-362) and the fused
// per-iteration step (train.cpp:402-475).  Host code: -ffp-contract=off.
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "primitives.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

constexpr int kMaxStepViews = 32;  // views per step between loss read-backs

struct Scratch {
    double ssim_sum;
    double l1_sum;
    unsigned long long skipped;
    uint32_t flags;
    uint32_t count;
    unsigned long long max_leak_bits;
    double leak_sum;
    double loss_acc;
    double pad[2];
    double view_sums[kMaxStepViews][2];  // per-view (ssim_sum, l1_sum) of a training step
    uint32_t abort;                      // sticky non-finite-loss flag of pipelined iterations
    uint32_t pad2;
    double pipe_sums[HGS_TRAIN_PIPELINE][kMaxStepViews][2];  // loss sums of pipelined iterations
    unsigned long long skipped_cum;  // rows skipped for non-finite gradients since upload / load
    double pipe_gate[HGS_TRAIN_PIPELINE][2];  // view-parallel: all-reduced sum of every rank's loss sums, 0
};

// sum of the n loss sums of a step (non-finite iff one of them is) -> gate[0], gate[1] = 0
__global__ void gate_sum_kernel(const double* __restrict__ sums, int n, double* __restrict__ gate) {
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) v += sums[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) {
        gate[0] = v;
        gate[1] = 0.0;
    }
}
static_assert(kMaxStepViews == 32, "hgs_pending_step::dims");

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
#define CKL()                                                                                         \
    do {                                                                                              \
        cudaError_t e_ = cudaGetLastError();                                                          \
        if (e_ != cudaSuccess)                                                                        \
            return fail(ctx, HGS_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

__global__ void f64_to_f32_kernel(const double* __restrict__ src, float* __restrict__ dst, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = (float)src[i];
}

// Host image (double or float) -> device float buffer, on stream s (default
// the context stream) with `stage` as the FP64 staging buffer.
hgs_status upload_image(hgs_ctx* ctx, const void* src, int dtype, int64_t n, DBuf& dst, cudaStream_t s = nullptr,
                        DBuf* stage = nullptr) {
    if (!s) s = ctx->stream;
    if (!stage) stage = &ctx->stage;
    if (dtype == HGS_U8) {  // 8-bit sRGB frame: stays 8-bit, decoded by the loss
        CK(dst.ensure((size_t)n));
        CK(cudaMemcpyAsync(dst.p, src, (size_t)n, cudaMemcpyHostToDevice, s));
        return HGS_OK;
    }
    CK(dst.ensure((size_t)n * 4));
    if (dtype == HGS_F32) {
        CK(cudaMemcpyAsync(dst.p, src, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    } else {
        CK(stage->ensure((size_t)n * 8));
        CK(cudaMemcpyAsync(stage->p, src, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        f64_to_f32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(stage->as<double>(), dst.as<float>(), n);
        count_launch();
        CKL();
    }
    return HGS_OK;
}

// The copy stream and the double-buffer events of the host-GT path.
hgs_status ensure_copy_stream(hgs_ctx* ctx) {
    if (ctx->copy_stream) return HGS_OK;
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        CK(cudaEventCreateWithFlags(&ctx->gt_ready[b], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->gt_free[b], cudaEventDisableTiming));
    }
    return HGS_OK;
}

hgs_status download_floats(hgs_ctx* ctx, const float* dev, int64_t n, void* host, int dtype) {
    if (dtype == HGS_F32) {
        CK(cudaMemcpyAsync(host, dev, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    } else {
        std::vector<float> tmp((size_t)n);
        CK(cudaMemcpyAsync(tmp.data(), dev, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int64_t i = 0; i < n; ++i) static_cast<double*>(host)[i] = tmp[(size_t)i];
    }
    return HGS_OK;
}

Scratch* scratch(hgs_ctx* ctx) { return ctx->scratch.as<Scratch>(); }

// The SSIM window and the sRGB LUT live in __constant__ memory, one copy per
// device: set once per device (contexts on several GPUs in one process).
void ensure_loss_tables(int device) {
    static std::atomic<uint64_t> done{0};
    const uint64_t bit = 1ull << (device & 63);
    if (done.load() & bit) return;
    static std::mutex m;
    std::lock_guard<std::mutex> g(m);
    if (done.load() & bit) return;
    set_ssim_window();
    set_srgb_lut();
    done.fetch_or(bit);
}

hgs_status ensure_scratch(hgs_ctx* ctx) {
    if (!ctx->scratch.p) {
        CK(ctx->scratch.ensure(sizeof(Scratch)));
        CK(cudaMemset(ctx->scratch.p, 0, sizeof(Scratch)));
    }
    CK(ctx->pinned.ensure(256 + sizeof(Scratch)));
    return HGS_OK;
}

// K6 + exact pixels + K7 for the current tape; dL/dimage in device `lg`.
// The zeroing of the backward's outputs (screen norms, per-splat
// accumulators); the training step issues it before the loss so that the
// kernel chain loss -> K6 -> K7 has no memset in it (programmatic launches).
// V_bound: an upper bound of the render's visible count (N before the render).
hgs_status zero_backward(hgs_ctx* ctx, int64_t V_bound) {
    cudaStream_t st = ctx->stream;
    CK(cudaMemsetAsync(ctx->sn4.p, 0, (size_t)ctx->cap4 * 4, st));
    CK(cudaMemsetAsync(ctx->sn3.p, 0, (size_t)ctx->cap3 * 4, st));
    if (V_bound == 0) return HGS_OK;
    CK(ctx->accum.ensure((size_t)V_bound * kAccStrideHost * sizeof(acc_t)));
    CK(cudaMemsetAsync(ctx->accum.p, 0, (size_t)V_bound * kAccStrideHost * sizeof(acc_t), st));
    return HGS_OK;
}

hgs_status run_backward(hgs_ctx* ctx, const float* lg, double scale, bool zeroed = false) {
    cudaStream_t st = ctx->stream;
    const int64_t V = ctx->V;
    if (!zeroed) {
        hgs_status r = zero_backward(ctx, (ctx->V == 0 || ctx->I == 0) ? 0 : ctx->V);
        if (r != HGS_OK) return r;
    }
    if (V == 0 || ctx->I == 0) return HGS_OK;
    const int n_tiles = ctx->tiles_x * ctx->tiles_y;
    prof_begin(ctx, PH_RASTER_BWD);
    const bool exact = ctx->exact_backward;
    if (exact) {
        // exact backward mode: every pixel through the FP64 walk with FP64
        // colours (hgs_set_exact_backward)
        CK(ctx->exact_col.ensure((size_t)V * 3 * sizeof(double)));
        CK(launch_pdl(exact_colour_kernel, dim3(div_up((uint32_t)V, 128)), dim3(128), 0, st, ctx->sorted_gid, (int)V,
                      (int)ctx->n4, ctx->p4.as<float>(), ctx->cap4, ctx->p3.as<float>(), ctx->cap3, ctx->deg, ctx->cam,
                      ctx->t, ctx->exact_col.as<double>()));
        count_launch();
        CKL();
    } else {
        // K6; the FP64 backward of each tile's fix-up pixels runs inside the
        // tile's CTA after its walk (exact_bwd_pixel, with the forward
        // fix-up's FP64 colour)
        CK(launch_pdl(raster_bwd_kernel, dim3(n_tiles), dim3(128), 0, st, ctx->ranges.as<uint2>(),
                      static_cast<const uint32_t*>(ctx->inst_vals_final), ctx->fast_sorted.as<SplatFast>(),
                      ctx->rec_sorted.as<SplatRec>(), ctx->W, ctx->H, ctx->tiles_x, ctx->tfinal.as<float>(),
                      ctx->last.as<uint32_t>(), lg, (float)ctx->bg[0], (float)ctx->bg[1], (float)ctx->bg[2],
                      ctx->accum.as<acc_t>(),
                      static_cast<const uint32_t*>(tile_order_enabled() ? ctx->tile_order.as<uint32_t>() : nullptr),
                      static_cast<const uint32_t*>(ctx->fix_slot.as<uint32_t>()),
                      static_cast<const double*>(ctx->fix_cout.as<double>()), ctx->bg[0], ctx->bg[1], ctx->bg[2]));
        count_launch();
        CKL();
    }
    if (exact) {
        CK(launch_pdl(raster_bwd_exact_kernel, dim3(ctx->sms * 8), dim3(128), 0, st, ctx->W * ctx->H,
                      ctx->ranges.as<uint2>(), ctx->inst_vals_final, ctx->rec_sorted.as<SplatRec>(), ctx->W,
                      ctx->tiles_x, ctx->bg[0], ctx->bg[1], ctx->bg[2], ctx->last.as<uint32_t>(), lg,
                      ctx->exact_col.as<double>(), ctx->accum.as<acc_t>()));
        count_launch();
        CKL();
    }
    prof_end(ctx);
    prof_begin(ctx, PH_GAUSS_BWD);
    const int N = (int)(ctx->n4 + ctx->n3);
    CK(ctx->ddir.ensure((size_t)N * sizeof(float4)));
    const int first = ctx->grads_zero ? 1 : 0;
    if (!exact) {
        CK(launch_pdl(sh_bwd_kernel, dim3(div_up((uint32_t)N, 128)), dim3(128), 0, st, N,
                      ctx->sorted_of_gid.as<uint32_t>(), ctx->accum.as<acc_t>(), kAccStrideHost, (int)ctx->n4,
                      ctx->p4.as<float>(), ctx->cap4, ctx->p3.as<float>(), ctx->cap3, ctx->deg, (float)scale, ctx->g4,
                      ctx->g3, ctx->shdir.as<ShRec>(), ctx->ddir.as<float4>(), first));
        count_launch();
        CKL();
    }
    CK(launch_pdl(exact ? gaussian_bwd_exact_kernel : gaussian_bwd_kernel, dim3(div_up((uint32_t)N, 128)), dim3(128),
                  0, st, N, ctx->sorted_of_gid.as<uint32_t>(), ctx->accum.as<acc_t>(), kAccStrideHost, (int)ctx->n4,
                  ctx->p4.as<float>(), ctx->cap4, ctx->p3.as<float>(), ctx->cap3, ctx->deg, ctx->cam, ctx->t, scale,
                  ctx->g4, ctx->g3, ctx->sn4.as<float>(), ctx->sn3.as<float>(), ctx->dgn4, ctx->dgn3, ctx->dcnt4,
                  ctx->dcnt3, &ctx->rec_sorted.as<SplatRec>()->c00, (int)(sizeof(SplatRec) / sizeof(double)),
                  ctx->ddir.as<float4>(), first));
    count_launch();
    CKL();
    ctx->grads_zero = false;
    prof_end(ctx);
    return HGS_OK;
}

// K5 on the last rendered image against device gt; writes ctx->lgrad and
// accumulates the loss into scratch->loss_acc (device) -- no host sync.
// sums (device, optional): where to accumulate (ssim_sum, l1_sum); default
// the scratch pair read by the loss API
// img / W / H: the rendered image (default: the context's last render)
hgs_status run_loss(hgs_ctx* ctx, const void* gt, bool gt_u8, double lambda, double* sums = nullptr,
                    bool sums_zeroed = false, const float* img = nullptr, int W = -1, int H = -1) {
    cudaStream_t st = ctx->stream;
    if (!img) img = ctx->img.as<float>();
    if (W < 0) W = ctx->W;
    if (H < 0) H = ctx->H;
    const bool with_ssim = lambda != 0.0;
    if (with_ssim && (W < 11 || H < 11))
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
    ensure_loss_tables(ctx->device);
    const size_t npx = (size_t)W * H;
    CK(ctx->lgrad.ensure(npx * 3 * 4));
    Scratch* sc = scratch(ctx);
    if (!sums) sums = &sc->ssim_sum;
    if (!sums_zeroed) CK(cudaMemsetAsync(sums, 0, 2 * sizeof(double), st));  // ssim_sum, l1_sum
    const int vw = W - 10, vh = H - 10;
    prof_begin(ctx, PH_LOSS);
    if (with_ssim) CK(ctx->loss_ws.ensure((size_t)vw * vh * 9 * 4));
    launch_loss(st, img, gt, gt_u8, W, H, ctx->loss_ws.as<float>(), (float)lambda, with_ssim,
                ctx->lgrad.as<float>(), sums);
    count_launch(with_ssim ? 2 : 1);
    CKL();
    prof_end(ctx);
    return HGS_OK;
}

double loss_from_sums(double ssim_sum, double l1_sum, int W, int H, double lambda) {
    // loss.cpp:26-32: (1-l) * L1 + l * (1 - SSIM)
    const double n = (double)W * H * 3;
    double loss = (1.0 - lambda) * (l1_sum / n);
    if (lambda != 0.0) loss += lambda * (1.0 - ssim_sum / ((double)(W - 10) * (H - 10) * 3));
    return loss;
}
double loss_from_sums(const Scratch& h, int W, int H, double lambda) {
    return loss_from_sums(h.ssim_sum, h.l1_sum, W, H, lambda);
}

// view_sums/n_views (device, optional): the step's per-view loss sums; the
// kernels leave every parameter untouched when one is non-finite (the step
// then fails with NumericAbort, train.cpp:445-447, without a host round trip
// before the update).
// Adam over the Gaussians [lo, hi) of each pool (hi < 0: to the end; lo a
// multiple of 4): the kernels see row pointers offset by lo and n = hi - lo
// (the row stride stays the capacity).  cumulative = false: the step's
// skipped count is not added to GradAccum::skipped_nonfinite here (the
// sharded exchange adds the all-reduced count).
hgs_status run_adam(hgs_ctx* ctx, const hgs_lrs* lrs, double mean_lr_scale, const double* view_sums = nullptr,
                    int n_views = 0, uint32_t* abort = nullptr, int64_t lo4 = 0, int64_t hi4 = -1, int64_t lo3 = 0,
                    int64_t hi3 = -1, bool cumulative = true) {
    if (hi4 < 0) hi4 = ctx->n4;
    if (hi3 < 0) hi3 = ctx->n3;
    cudaStream_t st = ctx->stream;
    ctx->step++;
    const double bc1 = 1.0 - std::pow(0.9, (double)ctx->step);
    const double bc2 = 1.0 - std::pow(0.999, (double)ctx->step);
    AdamArgs A;
    A.b1 = 0.9f;
    A.b2 = 0.999f;
    A.one_m_b1 = (float)(1.0 - 0.9);
    A.one_m_b2 = (float)(1.0 - 0.999);
    A.inv_bc1 = (float)(1.0 / bc1);
    A.inv_bc2 = (float)(1.0 / bc2);
    A.lr_mean = (float)(lrs->mean * ctx->extent * mean_lr_scale);  // train.cpp:137
    A.lr_mean_t = (float)(lrs->mean_t * mean_lr_scale);           // train.cpp:138
    A.lr_quat = (float)lrs->quat;
    A.lr_scales = (float)lrs->scales;
    A.lr_opacity = (float)lrs->opacity;
    A.lr_sh = (float)lrs->sh;
    A.view_sums = view_sums;
    A.n_views = n_views;
    A.abort = abort;
    const int n4 = (int)std::max<int64_t>(0, hi4 - lo4), n3 = (int)std::max<int64_t>(0, hi3 - lo3);
    const int n = n4 + n3;
    Scratch* sc = scratch(ctx);
    A.skipped_cum = cumulative ? &sc->skipped_cum : nullptr;
    AdamPools P;
    P.p4 = ctx->p4.as<float>() + lo4, P.g4 = ctx->g4 + lo4, P.m4 = ctx->m4.as<float>() + lo4,
    P.v4 = ctx->v4.as<float>() + lo4;
    P.p3 = ctx->p3.as<float>() + lo3, P.g3 = ctx->g3 + lo3, P.m3 = ctx->m3.as<float>() + lo3,
    P.v3 = ctx->v3.as<float>() + lo3;
    P.gn4 = ctx->gn4.as<float>() + lo4, P.cnt4 = ctx->cnt4.as<float>() + lo4, P.dgn4 = ctx->dgn4 + lo4,
    P.dcnt4 = ctx->dcnt4 + lo4;
    P.gn3 = ctx->gn3.as<float>() + lo3, P.cnt3 = ctx->cnt3.as<float>() + lo3, P.dgn3 = ctx->dgn3 + lo3,
    P.dcnt3 = ctx->dcnt3 + lo3;
    P.cap4 = ctx->cap4, P.cap3 = ctx->cap3, P.n4 = n4, P.n3 = n3, P.K3 = 3 * sh_count(ctx->deg);
    prof_begin(ctx, PH_ADAM);
    if (n > 0) {
        CK(ctx->adam_ok.ensure((size_t)(5 * ctx->cap3 + 7 * ctx->cap4)));
        uint8_t* ok3 = ctx->adam_ok.as<uint8_t>() + lo3;
        uint8_t* ok4 = ctx->adam_ok.as<uint8_t>() + 5 * ctx->cap3 + lo4;
        const uint32_t units = adam_class_units(n3, n4, P.K3);
        CK(launch_pdl(adam_classes_kernel, dim3(div_up(units, 128)), dim3(128), 0, st, P, A, ok3, ok4, &sc->skipped,
                      &sc->flags));
        count_launch();
        CKL();
        const int bpr3 = (int)div_up(div_up((uint32_t)n3, 4), 256), bpr4 = (int)div_up(div_up((uint32_t)n4, 4), 256);
        const int R3 = R3_SH + P.K3 - 4, R4 = R4_SH + P.K3 - 8;
        const int blocks = R3 * bpr3 + R4 * bpr4;
        if (blocks > 0) {
            CK(launch_pdl(adam_rows_kernel, dim3(blocks), dim3(256), 0, st, P, A, ok3, ok4, bpr3, bpr4));
            count_launch();
            CKL();
        }
    }
    // the update zeroes every gradient row (a gated-off update does not: the
    // NumericAbort paths clear the buffer themselves)
    ctx->grads_zero = true;
    prof_end(ctx);
    return HGS_OK;
}

}  // namespace

extern "C" {

hgs_status hgs_forward_train(hgs_ctx* ctx, const hgs_camera* cam, double t, const double bg[3],
                             const hgs_raster_opts* opts, float* rgb_host) {
    if (!ctx || !cam || !bg) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = hgs_render_pipeline(ctx, cam, t, bg, opts);
    if (r != HGS_OK) return r;
    if (rgb_host) {
        CK(cudaMemcpyAsync(rgb_host, ctx->img.p, (size_t)ctx->W * ctx->H * 12, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    return HGS_OK;
}

hgs_status hgs_backward(hgs_ctx* ctx, const void* loss_grad, int dtype, int on_device, double scale) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "backward: no forward_train tape on this context");
    CK(cudaSetDevice(ctx->device));
    const float* lg;
    const int64_t n = (int64_t)ctx->W * ctx->H * 3;
    if (on_device) {
        lg = loss_grad ? static_cast<const float*>(loss_grad) : ctx->lgrad.as<float>();
        if (!lg) return fail(ctx, HGS_ERR_STATE, "backward: no device loss gradient");
    } else {
        if (!loss_grad) return HGS_ERR_INVALID_ARGUMENT;
        hgs_status r = upload_image(ctx, loss_grad, dtype, n, ctx->lgrad);
        if (r != HGS_OK) return r;
        lg = ctx->lgrad.as<float>();
    }
    hgs_status r = run_backward(ctx, lg, scale);
    if (r != HGS_OK) return r;
    CK(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

hgs_status hgs_zero_grads(hgs_ctx* ctx) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (ctx->gbuf.p) CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
    ctx->grads_zero = ctx->gbuf.p != nullptr;
    return HGS_OK;
}

hgs_status hgs_grads_download(hgs_ctx* ctx, hgs_host_scene* out, int dtype, void* sn4, void* sn3) {
    if (!ctx || !out) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    // reuse the scene download path on the gradient rows
    DBuf p4 = ctx->p4, p3 = ctx->p3;
    ctx->p4.p = ctx->g4;
    ctx->p3.p = ctx->g3;
    hgs_status r = hgs_scene_download(ctx, out, dtype);
    ctx->p4 = p4;
    ctx->p3 = p3;
    if (r != HGS_OK) return r;
    if (sn4 && ctx->n4) {
        r = download_floats(ctx, ctx->sn4.as<float>(), ctx->n4, sn4, dtype);
        if (r != HGS_OK) return r;
    }
    if (sn3 && ctx->n3) {
        r = download_floats(ctx, ctx->sn3.as<float>(), ctx->n3, sn3, dtype);
        if (r != HGS_OK) return r;
    }
    return HGS_OK;
}

// Packed payload ([0, n) of every gradient row + stat deltas) for the
// multi-GPU all-reduce: pack = 0 -> device buffer filled from the gradient
// buffer (ptr/count returned), pack = 1 -> the buffer scattered back.
hgs_status hgs_grads_packed(hgs_ctx* ctx, int unpack, float** ptr, int64_t* count) {
    if (!ctx || (!unpack && (!ptr || !count))) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->gbuf.p) return fail(ctx, HGS_ERR_STATE, "grads_packed: no scene uploaded");
    CK(cudaSetDevice(ctx->device));
    const int r4 = rows4(ctx->deg), r3 = rows3(ctx->deg);
    const int64_t n = (int64_t)r4 * ctx->n4 + (int64_t)r3 * ctx->n3 + 2 * (ctx->n4 + ctx->n3);
    CK(ctx->gpack.ensure((size_t)std::max<int64_t>(n, 1) * 4));
    if (n > 0) {
        grads_pack_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
            ctx->gbuf.as<float>(), ctx->g3 - ctx->g4, ctx->dgn4 - ctx->g4, r4, r3, ctx->cap4, ctx->cap3,
            (int)ctx->n4, (int)ctx->n3, ctx->gpack.as<float>(), unpack);
        count_launch();
        CKL();
    }
    if (unpack) {
        ctx->grads_zero = false;
    } else {
        *ptr = ctx->gpack.as<float>();
        *count = n;
    }
    return HGS_OK;
}

hgs_status hgs_grads_device(hgs_ctx* ctx, float** ptr, int64_t* count) {
    if (!ctx || !ptr || !count) return HGS_ERR_INVALID_ARGUMENT;
    *ptr = ctx->gbuf.as<float>();
    *count = ctx->gbuf_floats;
    ctx->grads_zero = false;  // the caller may write into it (e.g. an in-place all-reduce)
    return HGS_OK;
}

hgs_status hgs_loss_with_grad(hgs_ctx* ctx, const void* gt, int dtype, int on_device, double lambda, double* loss_out,
                              void* grad_host_out) {
    if (!ctx || !gt) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "loss: render an image first");
    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    const int64_t n = (int64_t)ctx->W * ctx->H * 3;
    const float* g;
    if (on_device) {
        g = static_cast<const float*>(gt);
    } else {
        r = upload_image(ctx, gt, dtype, n, ctx->gt_stage);
        if (r != HGS_OK) return r;
        g = ctx->gt_stage.as<float>();
    }
    r = run_loss(ctx, g, false, lambda);
    if (r != HGS_OK) return r;
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    CK(cudaMemcpyAsync(h, ctx->scratch.p, sizeof(Scratch), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (loss_out) *loss_out = loss_from_sums(*h, ctx->W, ctx->H, lambda);
    if (grad_host_out) return download_floats(ctx, ctx->lgrad.as<float>(), n, grad_host_out, dtype);
    return HGS_OK;
}

// PSNR / SSIM of ctx->img (W x H) against a device frame (metrics.cpp:91-101)
hgs_status metrics_impl(hgs_ctx* ctx, const void* g, bool gt_u8, double* psnr_out, double* ssim_out) {
    const int W = ctx->W, H = ctx->H;
    ensure_loss_tables(ctx->device);
    const int64_t n = (int64_t)W * H * 3;
    Scratch* sc = scratch(ctx);
    CK(cudaMemsetAsync(sc, 0, 2 * sizeof(double), ctx->stream));
    if (W >= 11 && H >= 11) CK(ctx->loss_ws.ensure((size_t)(W - 10) * (H - 10) * 9 * 4));
    launch_metrics(ctx->stream, ctx->img.as<float>(), g, gt_u8, W, H, ctx->loss_ws.as<float>(), &sc->ssim_sum);
    count_launch(2);
    CKL();
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    CK(cudaMemcpyAsync(h, sc, 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    const double mse = h->l1_sum / (double)n;  // the squared-difference sum
    if (psnr_out) *psnr_out = mse == 0.0 ? INFINITY : 10.0 * std::log10(1.0 / mse);
    if (ssim_out) *ssim_out = h->ssim_sum / ((double)(W - 10) * (H - 10) * 3);
    return HGS_OK;
}

hgs_status hgs_image_metrics(hgs_ctx* ctx, const void* gt, int dtype, int on_device, double* psnr_out,
                             double* ssim_out) {
    if (!ctx || !gt) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->have_tape) return fail(ctx, HGS_ERR_STATE, "metrics: render an image first");
    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    if (ssim_out && (ctx->W < 11 || ctx->H < 11))  // metrics.cpp:38-39
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
    const void* g = gt;
    if (!on_device) {
        r = upload_image(ctx, gt, dtype, (int64_t)ctx->W * ctx->H * 3, ctx->gt_stage);
        if (r != HGS_OK) return r;
        g = ctx->gt_stage.p;
    } else if (dtype == HGS_F64) {
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "metrics: device frames are HGS_F32 or HGS_U8");
    }
    return metrics_impl(ctx, g, dtype == HGS_U8, psnr_out, ssim_out);
}

hgs_status hgs_metrics(hgs_ctx* ctx, const void* a, const void* b, int dtype, int width, int height,
                       double* psnr_out, double* ssim_out) {
    if (!ctx || !a || !b || width <= 0 || height <= 0 || dtype == HGS_U8) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    if (ssim_out && (width < 11 || height < 11))
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "ssim: images smaller than the 11x11 window");
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    const int64_t n = (int64_t)width * height * 3;
    r = upload_image(ctx, a, dtype, n, ctx->img);
    if (r != HGS_OK) return r;
    r = upload_image(ctx, b, dtype, n, ctx->gt_stage);
    if (r != HGS_OK) return r;
    ctx->W = width;
    ctx->H = height;
    ctx->have_tape = false;  // img no longer belongs to a render
    return metrics_impl(ctx, ctx->gt_stage.p, false, psnr_out, ssim_out);
}

hgs_status hgs_photometric_loss_with_grad(hgs_ctx* ctx, const void* rendered, const void* gt, int dtype, int width,
                                          int height, double lambda, double* loss_out, void* grad_out) {
    if (!ctx || !rendered || !gt || width <= 0 || height <= 0) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    const int64_t n = (int64_t)width * height * 3;
    // its own image buffer: the last render (the tape of a pending backward)
    // stays valid, as the reference's pure loss function leaves it
    r = upload_image(ctx, rendered, dtype, n, ctx->loss_img);
    if (r != HGS_OK) return r;
    r = upload_image(ctx, gt, dtype, n, ctx->gt_stage);
    if (r != HGS_OK) return r;
    r = run_loss(ctx, ctx->gt_stage.as<float>(), false, lambda, nullptr, false, ctx->loss_img.as<float>(), width,
                 height);
    if (r != HGS_OK) return r;
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    CK(cudaMemcpyAsync(h, ctx->scratch.p, sizeof(Scratch), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (loss_out) *loss_out = loss_from_sums(*h, width, height, lambda);
    if (grad_out) return download_floats(ctx, ctx->lgrad.as<float>(), n, grad_out, dtype);
    return HGS_OK;
}

hgs_status hgs_adam_step(hgs_ctx* ctx, const hgs_lrs* lrs, double mean_lr_scale, int64_t* skipped_out) {
    if (!ctx || !lrs) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    Scratch* sc = scratch(ctx);
    CK(cudaMemsetAsync(&sc->skipped, 0, sizeof(unsigned long long) + 8, ctx->stream));
    r = run_adam(ctx, lrs, mean_lr_scale);
    if (r != HGS_OK) return r;
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    CK(cudaMemcpyAsync(h, ctx->scratch.p, sizeof(Scratch), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (skipped_out) *skipped_out = (int64_t)h->skipped;
    if (h->flags & FLAG_NONUNIT_QUAT)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "UnitQuat: cannot normalize zero/non-finite quaternion");
    return HGS_OK;
}

hgs_status hgs_adam_state_download(hgs_ctx* ctx, hgs_host_scene* m, hgs_host_scene* v, int dtype, uint64_t* step) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (ctx->state_sharded) return fail(ctx, HGS_ERR_STATE, "adam_state_download: the Adam moments are sharded (hgs_gather_state on every rank first)");
    DBuf p4 = ctx->p4, p3 = ctx->p3;
    hgs_status r = HGS_OK;
    if (m) {
        ctx->p4 = ctx->m4;
        ctx->p3 = ctx->m3;
        r = hgs_scene_download(ctx, m, dtype);
        ctx->p4 = p4;
        ctx->p3 = p3;
        if (r != HGS_OK) return r;
    }
    if (v) {
        ctx->p4 = ctx->v4;
        ctx->p3 = ctx->v3;
        r = hgs_scene_download(ctx, v, dtype);
        ctx->p4 = p4;
        ctx->p3 = p3;
        if (r != HGS_OK) return r;
    }
    if (step) *step = ctx->step;
    return HGS_OK;
}

hgs_status hgs_adam_state_upload(hgs_ctx* ctx, const hgs_host_scene* m, const hgs_host_scene* v, int dtype,
                                 uint64_t step) {
    if (!ctx || !m || !v) return HGS_ERR_INVALID_ARGUMENT;
    if (m->n4 != ctx->n4 || m->n3 != ctx->n3 || v->n4 != ctx->n4 || v->n3 != ctx->n3)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "adam state: pool sizes differ from the scene");
    ctx->state_sharded = false;
    hgs_status r = hgs_upload_rows(ctx, m, dtype, ctx->m4.as<float>(), ctx->m3.as<float>());
    if (r != HGS_OK) return r;
    r = hgs_upload_rows(ctx, v, dtype, ctx->v4.as<float>(), ctx->v3.as<float>());
    if (r != HGS_OK) return r;
    ctx->step = step;
    return HGS_OK;
}

// Host gradients (the SceneGrads of optimizer_step(scene, grads, ...),
// train.hpp:68-69) into the device gradient rows; the densification-
// statistic deltas are cleared (an uploaded gradient carries none).
hgs_status hgs_grads_upload(hgs_ctx* ctx, const hgs_host_scene* g, int dtype) {
    if (!ctx || !g) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->gbuf.p) return fail(ctx, HGS_ERR_STATE, "grads_upload: no scene uploaded");
    if (g->n4 != ctx->n4 || g->n3 != ctx->n3 || g->sh_degree != ctx->deg)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "grads_upload: pool sizes / SH degree differ from the scene");
    CK(cudaSetDevice(ctx->device));
    CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
    hgs_status r = hgs_upload_rows(ctx, g, dtype, ctx->g4, ctx->g3);
    if (r != HGS_OK) return r;
    ctx->grads_zero = false;
    return HGS_OK;
}

// Densification statistics (GradAccum::grad_norm* / count*, optim.hpp:32-41)
// into the device (e.g. when training resumes from a checkpoint state).
hgs_status hgs_stats_upload(hgs_ctx* ctx, const double* gn4, const uint32_t* c4, const double* gn3,
                            const uint32_t* c3) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->gbuf.p) return fail(ctx, HGS_ERR_STATE, "stats_upload: no scene uploaded");
    CK(cudaSetDevice(ctx->device));
    const int64_t n4 = ctx->n4, n3 = ctx->n3;
    std::vector<float> a(n4, 0.f), b(n4, 0.f), c(n3, 0.f), d(n3, 0.f);
    for (int64_t i = 0; i < n4; ++i) {
        if (gn4) a[i] = (float)gn4[i];
        if (c4) b[i] = (float)c4[i];
    }
    for (int64_t i = 0; i < n3; ++i) {
        if (gn3) c[i] = (float)gn3[i];
        if (c3) d[i] = (float)c3[i];
    }
    if (n4) {
        CK(cudaMemcpy(ctx->gn4.p, a.data(), n4 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->cnt4.p, b.data(), n4 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(ctx->dgn4, 0, n4 * 4));
        CK(cudaMemset(ctx->dcnt4, 0, n4 * 4));
    }
    if (n3) {
        CK(cudaMemcpy(ctx->gn3.p, c.data(), n3 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->cnt3.p, d.data(), n3 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemset(ctx->dgn3, 0, n3 * 4));
        CK(cudaMemset(ctx->dcnt3, 0, n3 * 4));
    }
    return HGS_OK;
}

hgs_status hgs_stats_download(hgs_ctx* ctx, double* gn4, uint32_t* c4, double* gn3, uint32_t* c3) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    const int64_t n4 = ctx->n4, n3 = ctx->n3;
    std::vector<float> a(n4), b(n4), da(n4), db(n4), c(n3), d(n3), dc(n3), dd(n3);
    if (n4) {
        CK(cudaMemcpy(a.data(), ctx->gn4.p, n4 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), ctx->cnt4.p, n4 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(da.data(), ctx->dgn4, n4 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(db.data(), ctx->dcnt4, n4 * 4, cudaMemcpyDeviceToHost));
    }
    if (n3) {
        CK(cudaMemcpy(c.data(), ctx->gn3.p, n3 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(d.data(), ctx->cnt3.p, n3 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dc.data(), ctx->dgn3, n3 * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(dd.data(), ctx->dcnt3, n3 * 4, cudaMemcpyDeviceToHost));
    }
    for (int64_t i = 0; i < n4; ++i) {
        if (gn4) gn4[i] = (double)a[i] + (double)da[i];
        if (c4) c4[i] = (uint32_t)(b[i] + db[i]);
    }
    for (int64_t i = 0; i < n3; ++i) {
        if (gn3) gn3[i] = (double)c[i] + (double)dc[i];
        if (c3) c3[i] = (uint32_t)(d[i] + dd[i]);
    }
    return HGS_OK;
}

hgs_status hgs_sweep_convert(hgs_ctx* ctx, int64_t* moved_out, hgs_conversion_report* report) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (!(ctx->tau > 0.0)) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "is_static: tau must be positive");
    if (!ctx->pipeline.empty()) return fail(ctx, HGS_ERR_STATE, "sweep_convert: pipelined iterations pending");
    if (ctx->state_sharded) return fail(ctx, HGS_ERR_STATE, "sweep_convert: the Adam moments are sharded (hgs_gather_state on every rank first)");

    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    cudaStream_t st = ctx->stream;
    ctx->dens_planned = false;  // the sweep moves rows: a pending densify plan is stale
    const int n4 = (int)ctx->n4, n3 = (int)ctx->n3;
    hgs_conversion_report rep{0, 0.0, 0.0};
    if (n4 == 0) {
        if (report) *report = rep;
        return HGS_OK;
    }
    // s_star: smallest double with exp(s_star) > tau under the host libm
    // (scene.cpp:12 evaluates std::exp(s_t) > tau); the device then compares
    // s_t >= s_star, exact for every float s_t.
    const double tau = ctx->tau;
    double s = std::log(tau);
    while (!(std::exp(s) > tau)) s = std::nextafter(s, INFINITY);
    for (;;) {
        const double p = std::nextafter(s, -INFINITY);
        if (std::exp(p) > tau) s = p;
        else break;
    }
    CK(ctx->visflag.ensure((size_t)n4 * 4));
    CK(ctx->vispos.ensure((size_t)n4 * 4));
    CK(ctx->scan_ws.ensure(scan_workspace_bytes(n4) + 4096));
    Scratch* sc = scratch(ctx);
    CK(cudaMemsetAsync(sc, 0, sizeof(Scratch), st));
    uint32_t* mask = ctx->visflag.as<uint32_t>();
    uint32_t* pos = ctx->vispos.as<uint32_t>();
    convert_mask_kernel<<<div_up(n4, 256), 256, 0, st>>>(ctx->p4.as<float>(), ctx->cap4, n4, s, mask);
    count_launch();
    CKL();
    exclusive_scan_u32(mask, pos, n4, &sc->count, ctx->scan_ws.as<uint32_t>(), st);
    CKL();
    CK(ctx->stage.ensure((size_t)n4 * 8 + 64));
    convert_rows_kernel<<<div_up(n4, 128), 128, 0, st>>>(
        ctx->p4.as<float>(), ctx->m4.as<float>(), ctx->v4.as<float>(), ctx->cap4, n4, mask, pos, ctx->p3.as<float>(),
        ctx->m3.as<float>(), ctx->v3.as<float>(), ctx->cap3, n3, ctx->deg, ctx->stage.as<long long>(),
        &sc->max_leak_bits, &sc->leak_sum, &sc->flags);
    count_launch();
    CKL();
    // survivors: stable compaction of params and both moments
    const int R4 = rows4(ctx->deg);
    compact_survivors_kernel<<<div_up(n4, 256), 256, 0, st>>>(ctx->p4.as<float>(), ctx->p4_alt.as<float>(), R4,
                                                              ctx->cap4, n4, mask, pos);
    count_launch();
    compact_survivors_kernel<<<div_up(n4, 256), 256, 0, st>>>(ctx->m4.as<float>(), ctx->m4_alt.as<float>(), R4,
                                                              ctx->cap4, n4, mask, pos);
    count_launch();
    compact_survivors_kernel<<<div_up(n4, 256), 256, 0, st>>>(ctx->v4.as<float>(), ctx->v4_alt.as<float>(), R4,
                                                              ctx->cap4, n4, mask, pos);
    count_launch();
    CKL();
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    CK(cudaMemcpyAsync(h, sc, sizeof(Scratch), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint32_t cnt = h->count;
    if (h->flags & FLAG_DEGENERATE_ROT)
        return fail(ctx, HGS_ERR_DEGENERATE_ROTATION, "extract_spatial_rot: spatial block is singular");
    if (h->flags & FLAG_NOT_ROTATION)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "rot3_to_quat: input is not a rotation matrix");
    if (moved_out && cnt) CK(cudaMemcpy(moved_out, ctx->stage.p, (size_t)cnt * 8, cudaMemcpyDeviceToHost));
    std::swap(ctx->p4, ctx->p4_alt);
    std::swap(ctx->m4, ctx->m4_alt);
    std::swap(ctx->v4, ctx->v4_alt);
    ctx->n4 = n4 - (int64_t)cnt;
    ctx->n3 = n3 + (int64_t)cnt;
    // train.cpp:357-361: every densify statistic is reset; gradients are
    // already zero after the Adam step, cleared here for the new row map.
    CK(cudaMemsetAsync(ctx->gn4.p, 0, (size_t)ctx->cap4 * 4, st));
    CK(cudaMemsetAsync(ctx->cnt4.p, 0, (size_t)ctx->cap4 * 4, st));
    CK(cudaMemsetAsync(ctx->gn3.p, 0, (size_t)ctx->cap3 * 4, st));
    CK(cudaMemsetAsync(ctx->cnt3.p, 0, (size_t)ctx->cap3 * 4, st));
    CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, st));
    ctx->grads_zero = true;
    CK(cudaStreamSynchronize(st));
    ctx->have_tape = false;
    rep.count = cnt;
    double mx;
    std::memcpy(&mx, &h->max_leak_bits, 8);
    rep.max_leakage = cnt ? mx : 0.0;
    rep.mean_leakage = cnt ? h->leak_sum / (double)cnt : 0.0;
    if (report) *report = rep;
    return HGS_OK;
}

// pipelined != 0: enqueue only (hgs_train_step_async); the loss sums land in
// the iteration's slot and are read by hgs_train_collect.
hgs_status train_step_impl(hgs_ctx* ctx, int n_views, const hgs_camera* cams, const double* times,
                           const void* const* gt, int gt_dtype, int gt_on_device, int batch_total,
                           const hgs_train_opts* o, int apply_adam, double* loss_out, int pipelined = 0) {
    if (!ctx || n_views < 0 || (n_views && (!cams || !times || !gt)) || !o || batch_total <= 0)
        return HGS_ERR_INVALID_ARGUMENT;
    CK(cudaSetDevice(ctx->device));
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    if (!pipelined && !ctx->pipeline.empty())
        return fail(ctx, HGS_ERR_STATE, "train_step: pipelined iterations pending (hgs_train_collect first)");
    if (pipelined) {
        if ((int)ctx->pipeline.size() >= HGS_TRAIN_PIPELINE)
            return fail(ctx, HGS_ERR_STATE, "train_step_async: pipeline full (hgs_train_collect first)");
        // more than kMaxStepViews views: view v adds its loss sums into slot
        // v % kMaxStepViews (the loss is linear in the sums of equal-size views)
        for (int v = kMaxStepViews; v < n_views; ++v)
            if (cams[v].width != cams[v % kMaxStepViews].width || cams[v].height != cams[v % kMaxStepViews].height)
                return fail(ctx, HGS_ERR_INVALID_ARGUMENT,
                            "train_step_async: more than 32 views per iteration need equal image sizes");
        if (!ctx->pipe_ev[0])
            for (int k = 0; k < HGS_TRAIN_PIPELINE; ++k)
                CK(cudaEventCreateWithFlags(&ctx->pipe_ev[k], cudaEventDisableTiming));
        CK(ctx->pinned_pipe.ensure(sizeof(double) * (2 * kMaxStepViews + 1) * HGS_TRAIN_PIPELINE));
    }
    const int slot = ctx->pipe_next;
    hgs_raster_opts ro{o->weight_cutoff, 1, 0, 0};
    // No host round trip per view beyond the render's instance count: the
    // per-view loss sums stay on the device (read every kMaxStepViews views
    // and at the end), Adam checks their finiteness itself.
    double loss = 0.0;
    Scratch* sc = scratch(ctx);
    Scratch* h = static_cast<Scratch*>(ctx->pinned.p);
    int pending = 0;  // views whose loss sums are still on the device
    auto flush = [&]() -> hgs_status {
        CK(cudaMemcpyAsync(h->view_sums, sc->view_sums, sizeof(double) * 2 * pending, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        for (int k = 0; k < pending; ++k)
            loss += loss_from_sums(h->view_sums[k][0], h->view_sums[k][1], ctx->W, ctx->H, o->ssim_lambda);
        pending = 0;
        return HGS_OK;
    };
    if (!gt_on_device) {
        r = ensure_copy_stream(ctx);
        if (r != HGS_OK) return r;
    }
    if (apply_adam)  // here, not between the last backward kernel and Adam (programmatic launches)
        CK(cudaMemsetAsync(&sc->skipped, 0, sizeof(unsigned long long) + 8, ctx->stream));
    for (int v = 0; v < n_views; ++v) {
        const void* g = nullptr;
        const int b = v & 1;
        if (!gt_on_device) {
            // e2e path: the view's ground truth comes from host memory.  It is
            // copied on the copy stream into one of two buffers while the view
            // renders; the loss waits for it, the copy into the same buffer
            // two views later waits for that loss.
            CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->gt_free[b], 0));
            r = upload_image(ctx, gt[v], gt_dtype, (int64_t)cams[v].width * cams[v].height * 3, ctx->gt_buf[b],
                             ctx->copy_stream, &ctx->gt_stage64[b]);
            if (r != HGS_OK) return r;
            CK(cudaEventRecord(ctx->gt_ready[b], ctx->copy_stream));
            g = ctx->gt_buf[b].p;
        } else {
            g = gt[v];
        }
        // the zeroing of this view's loss sums and backward outputs goes
        // ahead of its render, so render -> loss -> backward is one chain of
        // adjacent kernels (programmatic launches)
        double* vsums = pipelined ? sc->pipe_sums[slot][v % kMaxStepViews] : sc->view_sums[pending];
        ZeroJobs zj;  // filled by the render's own fill launch
        if (!pipelined || v < kMaxStepViews) zj.add(vsums, 2 * sizeof(double));
        zj.add(ctx->sn4.p, (size_t)ctx->cap4 * 4);
        zj.add(ctx->sn3.p, (size_t)ctx->cap3 * 4);
        {
            const int64_t Nv = ctx->n4 + ctx->n3;  // bound of the visible count
            CK(ctx->accum.ensure((size_t)std::max<int64_t>(Nv, 1) * kAccStrideHost * sizeof(acc_t)));
            zj.add(ctx->accum.p, (size_t)Nv * kAccStrideHost * sizeof(acc_t));
        }
        r = hgs_render_pipeline(ctx, &cams[v], times[v], o->bg, &ro, 1, 0, nullptr, &zj);
        if (r != HGS_OK) return r;
        if (!gt_on_device) CK(cudaStreamWaitEvent(ctx->stream, ctx->gt_ready[b], 0));
        r = run_loss(ctx, g, gt_dtype == HGS_U8, o->ssim_lambda, vsums, true);
        if (r != HGS_OK) return r;
        if (!gt_on_device) CK(cudaEventRecord(ctx->gt_free[b], ctx->stream));
        ++pending;
        r = run_backward(ctx, ctx->lgrad.as<float>(), 1.0 / (double)batch_total, true);  // train.cpp:430-432
        if (r != HGS_OK) return r;
        if (!pipelined && pending == kMaxStepViews && v + 1 < n_views) {
            r = flush();
            if (r != HGS_OK) return r;
        }
    }
    if (!std::isfinite(loss) && apply_adam) {  // an earlier group of views already failed
        if (loss_out) *loss_out = loss;
        // drop the aborted step's gradients and statistic deltas (no Adam ran,
        // so the step counter is unchanged), as the abort path below does
        CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
        ctx->grads_zero = true;
        r = hgs_render_finish(ctx);
        if (r != HGS_OK) return r;
        return fail(ctx, HGS_ERR_NUMERIC_ABORT, "train: non-finite loss");  // train.cpp:445-447
    }
    const int gate = std::min(pending, kMaxStepViews);
    const uint64_t step_before = ctx->step;
    if (apply_adam) {  // (the skipped counter was zeroed before the views)
        r = run_adam(ctx, &o->lrs, o->mean_lr_scale, pipelined ? &sc->pipe_sums[slot][0][0] : &sc->view_sums[0][0],
                     gate, pipelined ? &sc->abort : nullptr);
        if (r != HGS_OK) return r;
    }
    if (pipelined) {
        hgs_pending_step ps;
        ps.slot = slot;
        ps.n_views = n_views;
        for (int v = 0; v < std::min(n_views, kMaxStepViews); ++v) {
            ps.dims[v][0] = cams[v].width;
            ps.dims[v][1] = cams[v].height;
        }
        ps.lambda = o->ssim_lambda;
        ps.adam = apply_adam != 0;
        ps.step_before = step_before;
        double* hp = static_cast<double*>(ctx->pinned_pipe.p) + (size_t)slot * kMaxStepViews * 2;
        CK(cudaMemcpyAsync(hp, sc->pipe_sums[slot], sizeof(double) * 2 * std::min(n_views, kMaxStepViews),
                           cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaEventRecord(ctx->pipe_ev[slot], ctx->stream));
        ctx->pipeline.push_back(ps);
        ctx->pipe_next = (slot + 1) % HGS_TRAIN_PIPELINE;
        ctx->stats_pending = true;
        prof_collect(ctx);
        return HGS_OK;
    }
    r = flush();
    if (r != HGS_OK) return r;
    r = hgs_render_finish(ctx);
    if (r != HGS_OK) return r;
    if (loss_out) *loss_out = loss;
    // without the update the caller owns the decision (e.g. after summing the
    // batch loss over ranks), so a non-finite loss is returned, not raised
    if (!std::isfinite(loss) && apply_adam) {
        {
            --ctx->step;  // the kernels skipped the update (and left the gradients)
            CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
            ctx->grads_zero = true;
        }
        return fail(ctx, HGS_ERR_NUMERIC_ABORT, "train: non-finite loss");  // train.cpp:445-447
    }
    prof_collect(ctx);
    return HGS_OK;
}

hgs_status hgs_train_step(hgs_ctx* ctx, int n_views, const hgs_camera* cams, const double* times,
                          const float* const* gt_device, int batch_total, const hgs_train_opts* o, int apply_adam,
                          double* loss_out) {
    return train_step_impl(ctx, n_views, cams, times, reinterpret_cast<const void* const*>(gt_device), HGS_F32, 1,
                           batch_total, o, apply_adam, loss_out);
}

hgs_status hgs_train_step_async(hgs_ctx* ctx, int n_views, const hgs_camera* cams, const double* times,
                                const void* const* gt, int dtype, int gt_on_device, int batch_total,
                                const hgs_train_opts* o, int apply_adam) {
    if (gt_on_device && dtype == HGS_F64)
        return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "train_step_async: device frames are HGS_F32 or HGS_U8");
    return train_step_impl(ctx, n_views, cams, times, gt, dtype, gt_on_device ? 1 : 0, batch_total, o, apply_adam,
                           nullptr, 1);
}

int hgs_train_pending(hgs_ctx* ctx) { return ctx ? (int)ctx->pipeline.size() : 0; }

// View-parallel completion of the iteration just enqueued with
// hgs_train_step_async(apply_adam = 0): all-reduce of the loss-sum gate and of
// the packed gradients over the context's communicator, then the gated Adam
// step -- all stream-ordered, no host synchronisation.
hgs_status hgs_train_exchange_async(hgs_ctx* ctx, const hgs_train_opts* o) {
    if (!ctx || !o) return HGS_ERR_INVALID_ARGUMENT;
    if (ctx->pipeline.empty() || ctx->pipeline.back().adam || ctx->pipeline.back().dist)
        return fail(ctx, HGS_ERR_STATE, "train_exchange_async: enqueue an iteration with apply_adam = 0 first");
    if (!ctx->comm) return fail(ctx, HGS_ERR_STATE, "train_exchange_async: call hgs_comm_init first");
    CK(cudaSetDevice(ctx->device));
    hgs_pending_step& ps = ctx->pipeline.back();
    Scratch* sc = scratch(ctx);
    double* gate = sc->pipe_gate[ps.slot];
    gate_sum_kernel<<<1, 32, 0, ctx->stream>>>(&sc->pipe_sums[ps.slot][0][0], 2 * std::min(ps.n_views, kMaxStepViews),
                                               gate);
    count_launch();
    CKL();
    hgs_status r = comm_allreduce_f64_dev(ctx, gate, 1);
    if (r != HGS_OK) return r;
    if (ctx->sharded) {
        // reduce-scatter -> Adam on this rank's shard -> all-gather (comm.cu)
        r = comm_reduce_scatter_grads(ctx);
        if (r != HGS_OK) return r;
        ps.step_before = ctx->step;
        int64_t lo4, hi4, lo3, hi3;
        hgs_shard_range(ctx->n4, ctx->comm_size, ctx->comm_rank, &lo4, &hi4);
        hgs_shard_range(ctx->n3, ctx->comm_size, ctx->comm_rank, &lo3, &hi3);
        r = run_adam(ctx, &o->lrs, o->mean_lr_scale, gate, 1, &sc->abort, lo4, hi4, lo3, hi3, false);
        if (r != HGS_OK) return r;
        r = comm_sharded_finish(ctx, &sc->skipped, &sc->skipped_cum);
        if (r != HGS_OK) return r;
    } else {
        r = hgs_allreduce_grads(ctx);
        if (r != HGS_OK) return r;
        ps.step_before = ctx->step;
        r = run_adam(ctx, &o->lrs, o->mean_lr_scale, gate, 1, &sc->abort);
        if (r != HGS_OK) return r;
    }
    ps.adam = true;
    ps.dist = true;
    double* hg = static_cast<double*>(ctx->pinned_pipe.p) + (size_t)HGS_TRAIN_PIPELINE * kMaxStepViews * 2;
    CK(cudaMemcpyAsync(&hg[ps.slot], gate, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaEventRecord(ctx->pipe_ev[ps.slot], ctx->stream));
    return HGS_OK;
}

hgs_status hgs_train_collect(hgs_ctx* ctx, double* loss_out) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (ctx->pipeline.empty()) return fail(ctx, HGS_ERR_STATE, "train_collect: no pipelined iteration pending");
    CK(cudaSetDevice(ctx->device));
    const hgs_pending_step p = ctx->pipeline.front();
    ctx->pipeline.pop_front();
    CK(cudaEventSynchronize(ctx->pipe_ev[p.slot]));
    const double* hp = static_cast<const double*>(ctx->pinned_pipe.p) + (size_t)p.slot * kMaxStepViews * 2;
    double loss = 0.0;
    for (int v = 0; v < std::min(p.n_views, kMaxStepViews); ++v) {
        // slot v holds the sums of views v, v + 32, ... (equal sizes): the
        // constant lambda * 1 of loss.cpp:26-32 once per view
        const int nv = (p.n_views - v + kMaxStepViews - 1) / kMaxStepViews;
        loss += loss_from_sums(hp[2 * v], hp[2 * v + 1], p.dims[v][0], p.dims[v][1], p.lambda) +
                (p.lambda != 0.0 ? p.lambda * (nv - 1) : 0.0);
    }
    if (loss_out) *loss_out = loss;
    // view-parallel steps: the decision is the all-reduced one (every rank's
    // views), identical on every rank
    const double* hg = static_cast<const double*>(ctx->pinned_pipe.p) + (size_t)HGS_TRAIN_PIPELINE * kMaxStepViews * 2;
    const bool bad = p.dist ? !std::isfinite(hg[p.slot]) : !std::isfinite(loss);
    if (bad && p.adam) {
        // the device skipped this update and every later pending one
        if (p.adam) ctx->step = p.step_before;
        ctx->pipeline.clear();
        ctx->pipe_next = 0;
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaMemsetAsync(&scratch(ctx)->abort, 0, sizeof(uint32_t), ctx->stream));
        // the skipped updates left gradients behind: start the next iteration from zero
        CK(cudaMemsetAsync(ctx->gbuf.p, 0, (size_t)ctx->gbuf_floats * 4, ctx->stream));
        ctx->grads_zero = true;
        CK(cudaStreamSynchronize(ctx->stream));
        return fail(ctx, HGS_ERR_NUMERIC_ABORT, "train: non-finite loss");  // train.cpp:445-447
    }
    if (ctx->pipeline.empty()) {
        hgs_status r = hgs_render_finish(ctx);
        if (r != HGS_OK) return r;
    }
    return HGS_OK;
}

hgs_status hgs_train_step_host(hgs_ctx* ctx, int n_views, const hgs_camera* cams, const double* times,
                               const void* const* gt_host, int dtype, int batch_total, const hgs_train_opts* o,
                               int apply_adam, double* loss_out) {
    return train_step_impl(ctx, n_views, cams, times, gt_host, dtype, 0, batch_total, o, apply_adam, loss_out);
}

}  // extern "C"

// GradAccum::skipped_nonfinite of the device state (checkpoint.cu, and the
// C ABI's hgs_skipped_nonfinite)
hgs_status hgs_skipped_total(hgs_ctx* ctx, uint64_t* get, const uint64_t* set) {
    hgs_status r = ensure_scratch(ctx);
    if (r != HGS_OK) return r;
    unsigned long long* d = &scratch(ctx)->skipped_cum;
    if (set) {
        const unsigned long long v = *set;
        CK(cudaMemcpyAsync(d, &v, 8, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    if (get) {
        unsigned long long v = 0;
        CK(cudaMemcpyAsync(&v, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *get = v;
    }
    return HGS_OK;
}

extern "C" hgs_status hgs_skipped_nonfinite(hgs_ctx* ctx, uint64_t* get, const uint64_t* set) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    return hgs_skipped_total(ctx, get, set);
}
