// gpu_backend.cpp -- the reference's hot-path functions (gpu_backend.hpp)
// over the C ABI of include/hgs_gpu.h.  Host glue only: every render,
// gradient, optimizer and conversion step runs in libhgs_gpu.so's sm_100a
// kernels.  The scene crosses the boundary as the reference's per-class
// double arrays (scene.hpp:13-59 <-> hgs_host_scene); the training loop keeps
// it device resident for the whole run (train.cpp:382-494).
#include "gpu_backend.hpp"

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "hgs/errors.hpp"
#include "hgs_gpu.h"

namespace HGS_GPU_NS {

namespace {

// ---- context and errors
struct Ctx {
    hgs_ctx* p = nullptr;
    uint64_t tape_token = 0;  // bumped by every forward_train on this context
    Ctx() {
        const char* d = std::getenv("HGS_DEVICE");
        if (hgs_ctx_create(d ? std::atoi(d) : 0, &p) != HGS_OK) throw std::runtime_error("hgs: no CUDA device");
    }
    ~Ctx() { hgs_ctx_destroy(p); }
};
Ctx& ctx() {
    thread_local Ctx c;  // one context per host thread
    return c;
}

// hgs_status -> the reference's exception types (errors.hpp:9-33)
void check(hgs_status s) {
    if (s == HGS_OK) return;
    const std::string m = hgs_last_error(ctx().p) ? hgs_last_error(ctx().p) : "hgs: error";
    switch (s) {
        case HGS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
        case HGS_ERR_DEGENERATE_TEMPORAL: throw DegenerateTemporalError(m);
        case HGS_ERR_DEGENERATE_ROTATION: throw DegenerateRotationError(m);
        case HGS_ERR_NUMERIC_ABORT: throw NumericAbort(m);
        case HGS_ERR_FORMAT: throw FormatError(m);
        case HGS_ERR_INTEGRITY: throw IntegrityError(m);
        case HGS_ERR_UNSUPPORTED_VERSION: throw UnsupportedVersionError(m);
        default: throw std::runtime_error(m);
    }
}

// ---- HybridScene <-> hgs_host_scene (per-class row-major doubles)
struct Soa {
    std::vector<double> mx, mt, ql, qr, ls4, op4, sh4, m3, q3, ls3, op3, sh3;
    hgs_host_scene view{};
    void bind(int64_t n4, int64_t n3, int deg, double tau, double extent, double duration) {
        view.n4 = n4;
        view.n3 = n3;
        view.sh_degree = deg;
        view.tau = tau;
        view.extent = extent;
        view.duration_seconds = duration;
        view.mean_x = mx.data();
        view.mean_t = mt.data();
        view.ql = ql.data();
        view.qr = qr.data();
        view.log_s4 = ls4.data();
        view.op4 = op4.data();
        view.sh4 = sh4.data();
        view.mean3 = m3.data();
        view.quat3 = q3.data();
        view.log_s3 = ls3.data();
        view.op3 = op3.data();
        view.sh3 = sh3.data();
    }
    void size(int64_t n4, int64_t n3, int deg) {
        const size_t K3 = 3 * (size_t)sh_coeff_count(deg);
        mx.assign(3 * n4, 0.0);
        mt.assign(n4, 0.0);
        ql.assign(4 * n4, 0.0);
        qr.assign(4 * n4, 0.0);
        ls4.assign(4 * n4, 0.0);
        op4.assign(n4, 0.0);
        sh4.assign(K3 * n4, 0.0);
        m3.assign(3 * n3, 0.0);
        q3.assign(4 * n3, 0.0);
        ls3.assign(3 * n3, 0.0);
        op3.assign(n3, 0.0);
        sh3.assign(K3 * n3, 0.0);
    }
};

Soa to_soa(const HybridScene& s) {
    Soa o;
    const int64_t n4 = (int64_t)s.dynamics.size(), n3 = (int64_t)s.statics.size();
    o.size(n4, n3, s.sh_degree);
    const int K = sh_coeff_count(s.sh_degree);
    for (int64_t i = 0; i < n4; ++i) {
        const Gaussian4D& g = s.dynamics[i];
        if ((int)g.color.coeffs.size() != K)
            throw std::invalid_argument("hgs: every Gaussian must carry the scene's SH degree");
        for (int k = 0; k < 3; ++k) o.mx[3 * i + k] = g.mean_x[k];
        o.mt[i] = g.mean_t;
        const double l[4] = {g.rot.left.w, g.rot.left.x, g.rot.left.y, g.rot.left.z};
        const double r[4] = {g.rot.right.w, g.rot.right.x, g.rot.right.y, g.rot.right.z};
        for (int k = 0; k < 4; ++k) {
            o.ql[4 * i + k] = l[k];
            o.qr[4 * i + k] = r[k];
            o.ls4[4 * i + k] = g.log_scales[k];
        }
        o.op4[i] = g.opacity_logit;
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) o.sh4[(i * K + k) * 3 + c] = g.color.coeffs[k][c];
    }
    for (int64_t i = 0; i < n3; ++i) {
        const Gaussian3D& g = s.statics[i];
        if ((int)g.color.coeffs.size() != K)
            throw std::invalid_argument("hgs: every Gaussian must carry the scene's SH degree");
        const double q[4] = {g.rot.w, g.rot.x, g.rot.y, g.rot.z};
        for (int k = 0; k < 3; ++k) {
            o.m3[3 * i + k] = g.mean[k];
            o.ls3[3 * i + k] = g.log_scales[k];
        }
        for (int k = 0; k < 4; ++k) o.q3[4 * i + k] = q[k];
        o.op3[i] = g.opacity_logit;
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) o.sh3[(i * K + k) * 3 + c] = g.color.coeffs[k][c];
    }
    o.bind(n4, n3, s.sh_degree, s.tau, s.extent, s.duration_seconds);
    return o;
}

// The device quaternions are unit and canonical (the Adam step renormalises
// them like renorm_quat, train.cpp:46-53): set the fields directly, as the
// reference's checkpoint reader does.
UnitQuat quat_of(const double* q) {
    UnitQuat u;
    u.w = q[0];
    u.x = q[1];
    u.y = q[2];
    u.z = q[3];
    return u;
}

void from_soa(const Soa& o, HybridScene& s) {
    const int64_t n4 = o.view.n4, n3 = o.view.n3;
    const int deg = o.view.sh_degree, K = sh_coeff_count(deg);
    s.sh_degree = deg;
    s.dynamics.assign(n4, Gaussian4D{});
    for (int64_t i = 0; i < n4; ++i) {
        Gaussian4D& g = s.dynamics[i];
        g.mean_x = Vec3(o.mx[3 * i], o.mx[3 * i + 1], o.mx[3 * i + 2]);
        g.mean_t = o.mt[i];
        g.rot.left = quat_of(&o.ql[4 * i]);
        g.rot.right = quat_of(&o.qr[4 * i]);
        g.log_scales = Vec4(o.ls4[4 * i], o.ls4[4 * i + 1], o.ls4[4 * i + 2], o.ls4[4 * i + 3]);
        g.opacity_logit = o.op4[i];
        g.color = SHColor(deg);
        for (int k = 0; k < K; ++k)
            g.color.coeffs[k] = Vec3(o.sh4[(i * K + k) * 3], o.sh4[(i * K + k) * 3 + 1], o.sh4[(i * K + k) * 3 + 2]);
    }
    s.statics.assign(n3, Gaussian3D{});
    for (int64_t i = 0; i < n3; ++i) {
        Gaussian3D& g = s.statics[i];
        g.mean = Vec3(o.m3[3 * i], o.m3[3 * i + 1], o.m3[3 * i + 2]);
        g.rot = quat_of(&o.q3[4 * i]);
        g.log_scales = Vec3(o.ls3[3 * i], o.ls3[3 * i + 1], o.ls3[3 * i + 2]);
        g.opacity_logit = o.op3[i];
        g.color = SHColor(deg);
        for (int k = 0; k < K; ++k)
            g.color.coeffs[k] = Vec3(o.sh3[(i * K + k) * 3], o.sh3[(i * K + k) * 3 + 1], o.sh3[(i * K + k) * 3 + 2]);
    }
}

// The device scene back into `s` (pool sizes may have changed on the device).
void download_scene(HybridScene& s) {
    int64_t n4 = 0, n3 = 0;
    int32_t deg = 0;
    check(hgs_scene_counts(ctx().p, &n4, &n3, &deg));
    Soa o;
    o.size(n4, n3, deg);
    o.bind(n4, n3, deg, s.tau, s.extent, s.duration_seconds);
    check(hgs_scene_download(ctx().p, &o.view, HGS_F64));
    from_soa(o, s);
}

void upload_scene(const HybridScene& s) {
    Soa o = to_soa(s);
    check(hgs_scene_upload(ctx().p, &o.view, HGS_F64));
}

hgs_camera to_cam(const Camera& c) {
    hgs_camera k{};
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    for (int i = 0; i < 9; ++i) k.rot[i] = c.rot(i / 3, i % 3);
    for (int i = 0; i < 3; ++i) k.trans[i] = c.trans[i];
    k.width = c.width;
    k.height = c.height;
    k.near_ = c.near;
    k.far_ = c.far;
    return k;
}

hgs_raster_opts to_opts(const RasterOpts& o) {
    return hgs_raster_opts{o.weight_cutoff, o.num_threads, o.count_map ? 1 : 0, o.transmittance_map ? 1 : 0};
}

RenderStats to_stats(const hgs_render_stats& s) {
    RenderStats r;
    r.culled_depth = (size_t)s.culled_depth;
    r.culled_offscreen = (size_t)s.culled_offscreen;
    r.culled_degenerate = (size_t)s.culled_degenerate;
    r.culled_temporal = (size_t)s.culled_temporal;
    r.degenerate_temporal = (size_t)s.degenerate_temporal;
    r.projected = (size_t)s.projected;
    return r;
}

// GradAccum (optim.hpp:32-41) <-> device Adam state + statistics.  The
// reference's AdamBuf rows are laid out like the scene's parameter classes.
struct StateSoa {
    Soa m, v;
};

void upload_state(const HybridScene& s, const GradAccum& a) {
    const size_t n3 = s.statics.size(), n4 = s.dynamics.size();
    const int deg = s.sh_degree;
    const size_t K3 = 3 * (size_t)sh_coeff_count(deg);
    if (a.statics.mean.m.size() != 3 * n3 || a.dynamics.mean_x.m.size() != 3 * n4)
        throw std::invalid_argument("hgs: optimizer state is not sized like the scene");
    StateSoa st;
    for (Soa* o : {&st.m, &st.v}) o->size((int64_t)n4, (int64_t)n3, deg);
    auto put = [](const AdamBuf& b, std::vector<double>& m, std::vector<double>& v) {
        m.assign(b.m.begin(), b.m.end());
        v.assign(b.v.begin(), b.v.end());
    };
    put(a.dynamics.mean_x, st.m.mx, st.v.mx);
    put(a.dynamics.mean_t, st.m.mt, st.v.mt);
    put(a.dynamics.quat_left, st.m.ql, st.v.ql);
    put(a.dynamics.quat_right, st.m.qr, st.v.qr);
    put(a.dynamics.scales, st.m.ls4, st.v.ls4);
    put(a.dynamics.opacity, st.m.op4, st.v.op4);
    put(a.dynamics.sh, st.m.sh4, st.v.sh4);
    put(a.statics.mean, st.m.m3, st.v.m3);
    put(a.statics.quat, st.m.q3, st.v.q3);
    put(a.statics.scales, st.m.ls3, st.v.ls3);
    put(a.statics.opacity, st.m.op3, st.v.op3);
    put(a.statics.sh, st.m.sh3, st.v.sh3);
    (void)K3;
    for (Soa* o : {&st.m, &st.v}) o->bind((int64_t)n4, (int64_t)n3, deg, s.tau, s.extent, s.duration_seconds);
    check(hgs_adam_state_upload(ctx().p, &st.m.view, &st.v.view, HGS_F64, a.step));
    check(hgs_stats_upload(ctx().p, a.grad_norm4.empty() ? nullptr : a.grad_norm4.data(),
                           a.count4.empty() ? nullptr : a.count4.data(),
                           a.grad_norm3.empty() ? nullptr : a.grad_norm3.data(),
                           a.count3.empty() ? nullptr : a.count3.data()));
    const uint64_t sk = a.skipped_nonfinite;
    check(hgs_skipped_nonfinite(ctx().p, nullptr, &sk));
}

void download_state(const HybridScene& s, GradAccum& a) {
    const size_t n3 = s.statics.size(), n4 = s.dynamics.size();
    const int deg = s.sh_degree;
    a.resize(n3, n4, 3 * (size_t)sh_coeff_count(deg));
    StateSoa st;
    for (Soa* o : {&st.m, &st.v}) {
        o->size((int64_t)n4, (int64_t)n3, deg);
        o->bind((int64_t)n4, (int64_t)n3, deg, s.tau, s.extent, s.duration_seconds);
    }
    uint64_t step = 0;
    check(hgs_adam_state_download(ctx().p, &st.m.view, &st.v.view, HGS_F64, &step));
    auto get = [](AdamBuf& b, const std::vector<double>& m, const std::vector<double>& v) {
        b.m = m;
        b.v = v;
    };
    get(a.dynamics.mean_x, st.m.mx, st.v.mx);
    get(a.dynamics.mean_t, st.m.mt, st.v.mt);
    get(a.dynamics.quat_left, st.m.ql, st.v.ql);
    get(a.dynamics.quat_right, st.m.qr, st.v.qr);
    get(a.dynamics.scales, st.m.ls4, st.v.ls4);
    get(a.dynamics.opacity, st.m.op4, st.v.op4);
    get(a.dynamics.sh, st.m.sh4, st.v.sh4);
    get(a.statics.mean, st.m.m3, st.v.m3);
    get(a.statics.quat, st.m.q3, st.v.q3);
    get(a.statics.scales, st.m.ls3, st.v.ls3);
    get(a.statics.opacity, st.m.op3, st.v.op3);
    get(a.statics.sh, st.m.sh3, st.v.sh3);
    a.step = step;
    check(hgs_stats_download(ctx().p, a.grad_norm4.data(), a.count4.data(), a.grad_norm3.data(), a.count3.data()));
    uint64_t sk = 0;
    check(hgs_skipped_nonfinite(ctx().p, &sk, nullptr));
    a.skipped_nonfinite = (size_t)sk;
}

hgs_lrs to_lrs(const LearningRates& l) {
    return hgs_lrs{l.mean, l.mean_final_ratio, l.mean_t, l.quat, l.scales, l.opacity, l.sh};
}

}  // namespace

// ---------------------------------------------------------------- rendering
RenderOutput rasterize(const HybridScene& scene, const Camera& cam, double t, const Vec3& background,
                       const RasterOpts& opts) {
    Soa o = to_soa(scene);
    const hgs_camera kc = to_cam(cam);
    const hgs_raster_opts ro = to_opts(opts);
    RenderOutput out;
    out.rgb = Image(cam.width, cam.height);
    if (opts.count_map) out.counts.assign(out.rgb.pixels(), 0u);
    if (opts.transmittance_map) out.transmittance.assign(out.rgb.pixels(), 1.0);
    const double bg[3] = {background[0], background[1], background[2]};
    hgs_render_stats st{};
    check(hgs_rasterize(ctx().p, &o.view, HGS_F64, &kc, t, bg, &ro, out.rgb.data.data(),
                        opts.count_map ? out.counts.data() : nullptr,
                        opts.transmittance_map ? out.transmittance.data() : nullptr, &st));
    out.stats = to_stats(st);
    return out;
}

std::vector<uint32_t> density_map(const HybridScene& scene, const Camera& cam, double t, bool dynamics_only,
                                  double weight_cutoff) {
    upload_scene(scene);
    const hgs_camera kc = to_cam(cam);
    std::vector<uint32_t> counts((size_t)cam.width * cam.height);
    check(hgs_density_map(ctx().p, &kc, t, dynamics_only ? 1 : 0, weight_cutoff, counts.data()));
    return counts;
}

// ---------------------------------------------------------------- forward / backward
Image forward_train(const HybridScene& scene, const Camera& cam, double t, const Vec3& background,
                    const RasterOpts& opts, Tape& tape) {
    upload_scene(scene);
    const hgs_camera kc = to_cam(cam);
    const hgs_raster_opts ro = to_opts(opts);
    const double bg[3] = {background[0], background[1], background[2]};
    std::vector<float> rgb((size_t)cam.width * cam.height * 3);
    check(hgs_forward_train(ctx().p, &kc, t, bg, &ro, rgb.data()));
    Image img(cam.width, cam.height);
    for (size_t i = 0; i < rgb.size(); ++i) img.data[i] = rgb[i];
    // the tape stays on the device; this object is its handle
    tape = Tape{};
    tape.width = cam.width;
    tape.height = cam.height;
    tape.time = t;
    tape.background = background;
    tape.final_trans.assign(1, (double)++ctx().tape_token);
    return img;
}

void backward(const HybridScene& scene, const Camera& cam, const Tape& tape, const Image& loss_grad,
              SceneGrads& grads) {
    (void)cam;
    if (tape.final_trans.size() != 1 || tape.final_trans[0] != (double)ctx().tape_token)
        throw std::invalid_argument("backward: the tape is not this thread's last forward_train");
    if (loss_grad.width != tape.width || loss_grad.height != tape.height)
        throw std::invalid_argument("backward: loss gradient size differs from the rendered image");
    if (grads.statics.size() != scene.statics.size() || grads.dynamics.size() != scene.dynamics.size())
        throw std::invalid_argument("backward: grads must be resize_like'd to the scene");
    check(hgs_zero_grads(ctx().p));
    check(hgs_backward(ctx().p, loss_grad.data.data(), HGS_F64, 0, 1.0));
    const int64_t n4 = (int64_t)scene.dynamics.size(), n3 = (int64_t)scene.statics.size();
    Soa g;
    g.size(n4, n3, scene.sh_degree);
    g.bind(n4, n3, scene.sh_degree, scene.tau, scene.extent, scene.duration_seconds);
    std::vector<double> sn4(n4), sn3(n3);
    check(hgs_grads_download(ctx().p, &g.view, HGS_F64, sn4.data(), sn3.data()));
    const int K = sh_coeff_count(scene.sh_degree);
    // backward.hpp:71-74: accumulate into the caller's grads
    for (int64_t i = 0; i < n4; ++i) {
        Grad4D& d = grads.dynamics[i];
        for (int k = 0; k < 3; ++k) d.mean_x[k] += g.mx[3 * i + k];
        d.mean_t += g.mt[i];
        for (int k = 0; k < 4; ++k) {
            d.quat_left[k] += g.ql[4 * i + k];
            d.quat_right[k] += g.qr[4 * i + k];
            d.log_scales[k] += g.ls4[4 * i + k];
        }
        d.opacity_logit += g.op4[i];
        if ((int)d.sh.size() != K) d.sh.assign(K, Vec3::Zero());
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) d.sh[k][c] += g.sh4[(i * K + k) * 3 + c];
        d.screen_norm += sn4[i];
    }
    for (int64_t i = 0; i < n3; ++i) {
        Grad3D& d = grads.statics[i];
        for (int k = 0; k < 3; ++k) {
            d.mean[k] += g.m3[3 * i + k];
            d.log_scales[k] += g.ls3[3 * i + k];
        }
        for (int k = 0; k < 4; ++k) d.quat[k] += g.q3[4 * i + k];
        d.opacity_logit += g.op3[i];
        if ((int)d.sh.size() != K) d.sh.assign(K, Vec3::Zero());
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) d.sh[k][c] += g.sh3[(i * K + k) * 3 + c];
        d.screen_norm += sn3[i];
    }
}

double photometric_loss_with_grad(const Image& rendered, const Image& gt, double ssim_lambda, Image& grad) {
    if (!rendered.same_shape(gt)) throw std::invalid_argument("photometric_loss: image shapes differ");
    grad = Image(rendered.width, rendered.height);
    double loss = 0.0;
    check(hgs_photometric_loss_with_grad(ctx().p, rendered.data.data(), gt.data.data(), HGS_F64, rendered.width,
                                         rendered.height, ssim_lambda, &loss, grad.data.data()));
    return loss;
}

// ---------------------------------------------------------------- optimizer / conversion
void optimizer_step(HybridScene& scene, const SceneGrads& grads, GradAccum& state, const LearningRates& lrs,
                    double mean_lr_scale) {
    const int64_t n4 = (int64_t)scene.dynamics.size(), n3 = (int64_t)scene.statics.size();
    if ((int64_t)grads.dynamics.size() != n4 || (int64_t)grads.statics.size() != n3)
        throw std::invalid_argument("optimizer_step: grads are not sized like the scene");
    upload_scene(scene);
    upload_state(scene, state);
    const int K = sh_coeff_count(scene.sh_degree);
    Soa g;
    g.size(n4, n3, scene.sh_degree);
    for (int64_t i = 0; i < n4; ++i) {
        const Grad4D& d = grads.dynamics[i];
        for (int k = 0; k < 3; ++k) g.mx[3 * i + k] = d.mean_x[k];
        g.mt[i] = d.mean_t;
        for (int k = 0; k < 4; ++k) {
            g.ql[4 * i + k] = d.quat_left[k];
            g.qr[4 * i + k] = d.quat_right[k];
            g.ls4[4 * i + k] = d.log_scales[k];
        }
        g.op4[i] = d.opacity_logit;
        for (int k = 0; k < K && k < (int)d.sh.size(); ++k)
            for (int c = 0; c < 3; ++c) g.sh4[(i * K + k) * 3 + c] = d.sh[k][c];
    }
    for (int64_t i = 0; i < n3; ++i) {
        const Grad3D& d = grads.statics[i];
        for (int k = 0; k < 3; ++k) {
            g.m3[3 * i + k] = d.mean[k];
            g.ls3[3 * i + k] = d.log_scales[k];
        }
        for (int k = 0; k < 4; ++k) g.q3[4 * i + k] = d.quat[k];
        g.op3[i] = d.opacity_logit;
        for (int k = 0; k < K && k < (int)d.sh.size(); ++k)
            for (int c = 0; c < 3; ++c) g.sh3[(i * K + k) * 3 + c] = d.sh[k][c];
    }
    g.bind(n4, n3, scene.sh_degree, scene.tau, scene.extent, scene.duration_seconds);
    check(hgs_grads_upload(ctx().p, &g.view, HGS_F64));
    const hgs_lrs l = to_lrs(lrs);
    int64_t skipped = 0;
    check(hgs_adam_step(ctx().p, &l, mean_lr_scale, &skipped));
    // the scene and the moments back (statistics are not touched by the step)
    std::vector<double> gn3 = state.grad_norm3, gn4 = state.grad_norm4;
    std::vector<uint32_t> c3 = state.count3, c4 = state.count4;
    download_scene(scene);
    download_state(scene, state);
    state.grad_norm3 = gn3;
    state.grad_norm4 = gn4;
    state.count3 = c3;
    state.count4 = c4;
}

ConversionReport sweep_convert(HybridScene& scene, std::vector<std::size_t>* moved) {
    upload_scene(scene);
    std::vector<int64_t> mv(std::max<size_t>(scene.dynamics.size(), 1));
    hgs_conversion_report rep{};
    check(hgs_sweep_convert(ctx().p, mv.data(), &rep));
    download_scene(scene);
    if (moved) moved->assign(mv.begin(), mv.begin() + rep.count);
    ConversionReport r;
    r.count = (size_t)rep.count;
    r.max_leakage = rep.max_leakage;
    r.mean_leakage = rep.mean_leakage;
    return r;
}

// ---------------------------------------------------------------- training (train.cpp:366-494)
TrainResult train(const MultiViewDataset& dataset, const TrainConfig& cfg) {
    if (dataset.cameras.empty() || dataset.total_frames() == 0)
        throw std::invalid_argument("train: dataset is empty");
    // init_scene (data_io.cpp:189-238) on the device: GPU 3-NN
    const size_t n = dataset.init_points.size();
    std::vector<double> pos(3 * n), rgb(3 * n);
    for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
            pos[3 * i + k] = dataset.init_points[i].position[k];
            rgb[3 * i + k] = dataset.init_points[i].rgb[k];
        }
    const hgs_init_cfg ic{cfg.sh_degree, cfg.tau, dataset.duration_seconds, cfg.init_temporal_scale,
                          cfg.init_opacity};
    check(hgs_init_scene(ctx().p, pos.data(), rgb.data(), (int64_t)n, &ic));
    HybridScene scene;
    scene.tau = cfg.tau;
    scene.duration_seconds = dataset.duration_seconds;
    int64_t n4 = 0, n3 = 0;
    int32_t deg = 0;
    check(hgs_scene_counts(ctx().p, &n4, &n3, &deg));
    // the extent the device computed travels with the downloaded scene
    {
        Soa o;
        o.size(n4, n3, deg);
        o.bind(n4, n3, deg, scene.tau, 1.0, scene.duration_seconds);
        check(hgs_scene_download(ctx().p, &o.view, HGS_F64));
        from_soa(o, scene);
        scene.extent = o.view.extent;
    }
    GradAccum state;
    state.resize(scene.statics.size(), scene.dynamics.size(), 3 * (size_t)sh_coeff_count(scene.sh_degree));
    return HGS_GPU_NS::train_scene(std::move(scene), std::move(state), dataset, cfg);
}

TrainResult train_scene(HybridScene scene, GradAccum state, const MultiViewDataset& dataset, const TrainConfig& cfg) {
    cfg.validate();
    if (dataset.cameras.empty() || dataset.total_frames() == 0)
        throw std::invalid_argument("train: dataset is empty");
    TrainResult result;
    scene.tau = cfg.tau;
    upload_scene(scene);
    upload_state(scene, state);
    hgs_rng* rng = nullptr;  // the loop's std::mt19937_64(cfg.seed), shared by batches and densification
    check(hgs_rng_create(cfg.seed, &rng));
    struct RngGuard {
        hgs_rng* r;
        ~RngGuard() { hgs_rng_destroy(r); }
    } guard{rng};

    std::vector<std::pair<size_t, size_t>> samples;  // (camera, frame), train.cpp:390-392
    for (size_t c = 0; c < dataset.frames.size(); ++c)
        for (size_t f = 0; f < dataset.frames[c].size(); ++f) samples.emplace_back(c, f);
    std::vector<hgs_camera> cams;
    for (const Camera& c : dataset.cameras) cams.push_back(to_cam(c));
    const size_t probe_cam = 0, probe_frame = dataset.frames[0].size() / 2;

    hgs_train_opts o{};
    o.ssim_lambda = cfg.ssim_lambda;
    o.weight_cutoff = cfg.weight_cutoff;
    o.lrs = to_lrs(cfg.lrs);
    for (int k = 0; k < 3; ++k) o.bg[k] = dataset.background[k];
    const hgs_raster_opts ro{cfg.weight_cutoff, 1, 0, 0};
    const int B = cfg.batch_size;
    std::vector<uint64_t> pick((size_t)B);
    std::vector<hgs_camera> bc((size_t)B);
    std::vector<double> bt((size_t)B);
    std::vector<const void*> bg((size_t)B);
    const auto t0 = std::chrono::steady_clock::now();
    for (int iter = 1; iter <= cfg.iterations; ++iter) {
        check(hgs_rng_batch(rng, samples.size(), B, pick.data()));  // train.cpp:403-404
        for (int b = 0; b < B; ++b) {
            const auto [ci, fi] = samples[pick[b]];
            bc[b] = cams[ci];
            bt[b] = dataset.frames[ci][fi].time;
            bg[b] = dataset.frames[ci][fi].image.data.data();
        }
        o.mean_lr_scale = std::pow(cfg.lrs.mean_final_ratio, double(iter) / double(cfg.iterations));  // :449
        // renders, losses, backward scaled by 1/B, statistics, Adam (train.cpp:405-450)
        double loss = 0.0;
        const hgs_status s = hgs_train_step_host(ctx().p, B, bc.data(), bt.data(), bg.data(), HGS_F64, B, &o, 1, &loss);
        if (s == HGS_ERR_NUMERIC_ABORT)
            throw NumericAbort("train: non-finite loss at iteration " + std::to_string(iter));  // :446-447
        check(s);
        TrainLogRow row;
        row.iter = iter;
        row.loss = loss / double(B);
        if (iter >= cfg.warmup_iters && iter % cfg.densify_interval == 0) {
            if (iter <= cfg.densify_stop_iter) {  // :457-465
                const hgs_densify_cfg dc{cfg.grad_threshold, cfg.opacity_prune_eps, cfg.clone_size_frac,
                                         cfg.split_factor, (int64_t)cfg.max_gaussians};
                hgs_densify_report rep{};
                check(hgs_densify_and_prune(ctx().p, &dc, rng, &rep));
                if (cfg.opacity_reset_enabled && cfg.opacity_reset_interval > 0 &&
                    iter % cfg.opacity_reset_interval == 0)
                    check(hgs_opacity_reset(ctx().p, std::log(0.01 / 0.99)));
            }
            if (cfg.conversion_enabled) {  // :466-472 (Adam rows remapped on the device)
                hgs_conversion_report rep{};
                check(hgs_sweep_convert(ctx().p, nullptr, &rep));
                row.conversions = (size_t)rep.count;
            }
        }
        if (cfg.probe_interval > 0 && (iter % cfg.probe_interval == 0 || iter == cfg.iterations)) {  // :476-482
            const Frame& pf = dataset.frames[probe_cam][probe_frame];
            check(hgs_render(ctx().p, &cams[probe_cam], pf.time, o.bg, &ro, nullptr, nullptr, nullptr, nullptr));
            check(hgs_image_metrics(ctx().p, pf.image.data.data(), HGS_F64, 0, &row.probe_psnr, nullptr));
        }
        int64_t n4 = 0, n3 = 0;
        int32_t deg = 0;
        check(hgs_scene_counts(ctx().p, &n4, &n3, &deg));
        row.n_static = (size_t)n3;
        row.n_dynamic = (size_t)n4;
        row.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        result.log.rows.push_back(row);
    }
    download_scene(scene);
    download_state(scene, state);
    result.scene = std::move(scene);
    result.state = std::move(state);
    return result;
}

}  // namespace HGS_GPU_NS
