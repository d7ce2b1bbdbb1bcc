// ref_capi.cpp -- a C ABI over the REFERENCE library itself (compiled from
// /root/reference/proj/src against oracle/ref_shim), in the oracle's struct
// types (hgs_oracle.h), so the tests can run the reference's own code on
// the oracle's fixtures and pin the oracle against it.  TEST INFRASTRUCTURE
// ONLY: built into oracle/_ref/ by oracle/Makefile (target `ref`), never
// linked into the product.
//
// Each entry converts the SoA FP64 scene to the reference's AoS
// HybridScene (scene.hpp:13-59), calls the reference function named in its
// comment and converts the result back.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hgs/backward.hpp"
#include "hgs/data_io.hpp"
#include "hgs/errors.hpp"
#include "hgs/loss.hpp"
#include "hgs/raster.hpp"
#include "hgs/scene.hpp"
#include "hgs/train.hpp"
#include "hgs_oracle.h"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const hgs::DegenerateTemporalError*>(&e)) return HGSO_DEGENERATE_TEMPORAL;
    if (dynamic_cast<const hgs::DegenerateRotationError*>(&e)) return HGSO_DEGENERATE_ROTATION;
    if (dynamic_cast<const hgs::NumericAbort*>(&e)) return HGSO_NUMERIC_ABORT;
    return HGSO_INVALID_ARGUMENT;
}

// The quaternion fields are set directly, as the reference's own checkpoint
// reader does (data_io.cpp get_quat): the reference computes on exactly the
// values the oracle (and the FP32 device pools) hold.  The UnitQuat
// constructor would renormalise them (gauss_math.cpp:27-33) -- a 1e-8-level
// change for FP32-rounded unit quaternions, covered separately by the tests
// with quaternions normalised in FP64.
int g_quat_ctor = 0;  // hgsr_set_quat_ctor: build quaternions through UnitQuat's constructor

hgs::UnitQuat quat(const double* q) {
    if (g_quat_ctor) return hgs::UnitQuat(q[0], q[1], q[2], q[3]);
    hgs::UnitQuat u;
    u.w = q[0];
    u.x = q[1];
    u.y = q[2];
    u.z = q[3];
    return u;
}

hgs::SHColor sh(const double* c, int deg) {
    hgs::SHColor s(deg);
    for (int k = 0; k < hgs::sh_coeff_count(deg); ++k) s.coeffs[k] = hgs::Vec3(c[3 * k], c[3 * k + 1], c[3 * k + 2]);
    return s;
}

hgs::HybridScene to_scene(const hgso_scene& s) {
    hgs::HybridScene out;
    out.tau = s.tau;
    out.extent = s.extent;
    out.sh_degree = s.sh_degree;
    const int K3 = 3 * hgs::sh_coeff_count(s.sh_degree);
    out.dynamics.resize(s.n4);
    for (int64_t i = 0; i < s.n4; ++i) {
        hgs::Gaussian4D& g = out.dynamics[i];
        g.mean_x = hgs::Vec3(s.mean_x[3 * i], s.mean_x[3 * i + 1], s.mean_x[3 * i + 2]);
        g.mean_t = s.mean_t[i];
        g.rot.left = quat(s.ql + 4 * i);
        g.rot.right = quat(s.qr + 4 * i);
        g.log_scales = hgs::Vec4(s.log_s4[4 * i], s.log_s4[4 * i + 1], s.log_s4[4 * i + 2], s.log_s4[4 * i + 3]);
        g.opacity_logit = s.op4[i];
        g.color = sh(s.sh4 + K3 * i, s.sh_degree);
    }
    out.statics.resize(s.n3);
    for (int64_t i = 0; i < s.n3; ++i) {
        hgs::Gaussian3D& g = out.statics[i];
        g.mean = hgs::Vec3(s.mean3[3 * i], s.mean3[3 * i + 1], s.mean3[3 * i + 2]);
        g.rot = quat(s.quat3 + 4 * i);
        g.log_scales = hgs::Vec3(s.log_s3[3 * i], s.log_s3[3 * i + 1], s.log_s3[3 * i + 2]);
        g.opacity_logit = s.op3[i];
        g.color = sh(s.sh3 + K3 * i, s.sh_degree);
    }
    return out;
}

// Writes the pools back (the caller sized the arrays for the new counts).
void from_scene(const hgs::HybridScene& h, hgso_scene& s) {
    const int K = hgs::sh_coeff_count(s.sh_degree);
    s.n4 = (int64_t)h.dynamics.size();
    s.n3 = (int64_t)h.statics.size();
    for (int64_t i = 0; i < s.n4; ++i) {
        const hgs::Gaussian4D& g = h.dynamics[i];
        for (int k = 0; k < 3; ++k) s.mean_x[3 * i + k] = g.mean_x[k];
        s.mean_t[i] = g.mean_t;
        const double ql[4] = {g.rot.left.w, g.rot.left.x, g.rot.left.y, g.rot.left.z};
        const double qr[4] = {g.rot.right.w, g.rot.right.x, g.rot.right.y, g.rot.right.z};
        for (int k = 0; k < 4; ++k) {
            s.ql[4 * i + k] = ql[k];
            s.qr[4 * i + k] = qr[k];
            s.log_s4[4 * i + k] = g.log_scales[k];
        }
        s.op4[i] = g.opacity_logit;
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) s.sh4[(i * K + k) * 3 + c] = g.color.coeffs[k][c];
    }
    for (int64_t i = 0; i < s.n3; ++i) {
        const hgs::Gaussian3D& g = h.statics[i];
        const double q[4] = {g.rot.w, g.rot.x, g.rot.y, g.rot.z};
        for (int k = 0; k < 3; ++k) {
            s.mean3[3 * i + k] = g.mean[k];
            s.log_s3[3 * i + k] = g.log_scales[k];
        }
        for (int k = 0; k < 4; ++k) s.quat3[4 * i + k] = q[k];
        s.op3[i] = g.opacity_logit;
        for (int k = 0; k < K; ++k)
            for (int c = 0; c < 3; ++c) s.sh3[(i * K + k) * 3 + c] = g.color.coeffs[k][c];
    }
}

hgs::Camera to_cam(const hgso_camera& c) {
    hgs::Camera k;
    k.fx = c.fx;
    k.fy = c.fy;
    k.cx = c.cx;
    k.cy = c.cy;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) k.rot(i, j) = c.rot[3 * i + j];
    k.trans = hgs::Vec3(c.trans[0], c.trans[1], c.trans[2]);
    k.width = c.width;
    k.height = c.height;
    k.near = c.near_;
    k.far = c.far_;
    return k;
}

void put_stats(const hgs::RenderStats& r, hgso_stats* s) {
    if (!s) return;
    s->culled_depth = (int64_t)r.culled_depth;
    s->culled_offscreen = (int64_t)r.culled_offscreen;
    s->culled_degenerate = (int64_t)r.culled_degenerate;
    s->culled_temporal = (int64_t)r.culled_temporal;
    s->degenerate_temporal = (int64_t)r.degenerate_temporal;
    s->projected = (int64_t)r.projected;
}

hgs::Image to_image(const double* p, int w, int h) {
    hgs::Image img(w, h);
    std::memcpy(img.data.data(), p, sizeof(double) * img.data.size());
    return img;
}

}  // namespace

extern "C" {

const char* hgsr_last_error(void) { return g_err.c_str(); }
void hgsr_set_quat_ctor(int on) { g_quat_ctor = on; }

// rasterize (raster.hpp:79-80)
int hgsr_rasterize(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3], double cutoff,
                   int num_threads, double* rgb_out, uint32_t* count_out, double* trans_out, hgso_stats* stats) {
    try {
        hgs::RasterOpts o;
        o.weight_cutoff = cutoff;
        o.num_threads = num_threads;
        o.count_map = count_out != nullptr;
        o.transmittance_map = trans_out != nullptr;
        const hgs::RenderOutput r =
            hgs::rasterize(to_scene(*s), to_cam(*cam), t, hgs::Vec3(bg[0], bg[1], bg[2]), o);
        std::memcpy(rgb_out, r.rgb.data.data(), sizeof(double) * r.rgb.data.size());
        if (count_out) std::memcpy(count_out, r.counts.data(), sizeof(uint32_t) * r.counts.size());
        if (trans_out) std::memcpy(trans_out, r.transmittance.data(), sizeof(double) * r.transmittance.size());
        put_stats(r.stats, stats);
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// project_scene (raster.hpp:74-76): the splats in the reference's order
int hgsr_project_scene(const hgso_scene* s, const hgso_camera* cam, double t, double cutoff, hgso_splat* out,
                       int64_t cap, int64_t* n_out, hgso_stats* stats) {
    try {
        hgs::RenderStats st;
        const hgs::Camera c = to_cam(*cam);
        const std::vector<hgs::SplatPrimitive> v = hgs::project_scene(to_scene(*s), c, t, cutoff, &st);
        *n_out = (int64_t)v.size();
        put_stats(st, stats);
        if ((int64_t)v.size() > cap) return HGSO_OK;
        for (size_t i = 0; i < v.size(); ++i) {
            const hgs::SplatPrimitive& p = v[i];
            hgso_splat& o = out[i];
            std::memset(&o, 0, sizeof(o));
            o.sx = p.screen_mean[0];
            o.sy = p.screen_mean[1];
            o.conic[0] = p.conic(0, 0);
            o.conic[1] = p.conic(0, 1);
            o.conic[2] = p.conic(1, 0);
            o.conic[3] = p.conic(1, 1);
            o.depth = p.depth;
            for (int k = 0; k < 3; ++k) o.rgb[k] = p.rgb[k];
            o.alpha = p.alpha;
            o.radius = p.radius;
            o.pool = p.source_pool;
            o.index = (int32_t)p.source_index;
            o.gid = p.source_pool == 1 ? (int32_t)p.source_index : (int32_t)(s->n4 + p.source_index);
            const hgs::SplatBounds b = hgs::splat_bounds(p, c.width, c.height);
            o.x0 = b.x0;
            o.x1 = b.x1;
            o.y0 = b.y0;
            o.y1 = b.y1;
            const float df = (float)p.depth;
            std::memcpy(&o.depth_bits, &df, 4);
        }
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// forward_train + backward (backward.hpp:68-74): the image and the gradients
// (grads are accumulated into, like the reference's out-parameter)
int hgsr_forward_backward(const hgso_scene* s, const hgso_camera* cam, double t, const double bg[3], double cutoff,
                          const double* loss_grad, double* rgb_out, hgso_grads* g) {
    try {
        const hgs::HybridScene scene = to_scene(*s);
        const hgs::Camera c = to_cam(*cam);
        hgs::RasterOpts o;
        o.weight_cutoff = cutoff;
        hgs::Tape tape;
        const hgs::Image img = hgs::forward_train(scene, c, t, hgs::Vec3(bg[0], bg[1], bg[2]), o, tape);
        std::memcpy(rgb_out, img.data.data(), sizeof(double) * img.data.size());
        if (!loss_grad || !g) return HGSO_OK;
        hgs::SceneGrads gr;
        gr.resize_like(scene);
        hgs::backward(scene, c, tape, to_image(loss_grad, c.width, c.height), gr);
        const int K = hgs::sh_coeff_count(s->sh_degree);
        for (int64_t i = 0; i < s->n4; ++i) {
            const hgs::Grad4D& d = gr.dynamics[i];
            for (int k = 0; k < 3; ++k) g->mean_x[3 * i + k] += d.mean_x[k];
            g->mean_t[i] += d.mean_t;
            for (int k = 0; k < 4; ++k) {
                g->ql[4 * i + k] += d.quat_left[k];
                g->qr[4 * i + k] += d.quat_right[k];
                g->log_s4[4 * i + k] += d.log_scales[k];
            }
            g->op4[i] += d.opacity_logit;
            for (int k = 0; k < K; ++k)
                for (int cc = 0; cc < 3; ++cc) g->sh4[(i * K + k) * 3 + cc] += d.sh[k][cc];
            g->screen_norm4[i] += d.screen_norm;
        }
        for (int64_t i = 0; i < s->n3; ++i) {
            const hgs::Grad3D& d = gr.statics[i];
            for (int k = 0; k < 3; ++k) {
                g->mean3[3 * i + k] += d.mean[k];
                g->log_s3[3 * i + k] += d.log_scales[k];
            }
            for (int k = 0; k < 4; ++k) g->quat3[4 * i + k] += d.quat[k];
            g->op3[i] += d.opacity_logit;
            for (int k = 0; k < K; ++k)
                for (int cc = 0; cc < 3; ++cc) g->sh3[(i * K + k) * 3 + cc] += d.sh[k][cc];
            g->screen_norm3[i] += d.screen_norm;
        }
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// photometric_loss_with_grad (loss.hpp:12-13)
double hgsr_photometric_loss_with_grad(const double* a, const double* b, int w, int h, double lambda, double* grad) {
    hgs::Image g;
    const double l = hgs::photometric_loss_with_grad(to_image(a, w, h), to_image(b, w, h), lambda, g);
    std::memcpy(grad, g.data.data(), sizeof(double) * g.data.size());
    return l;
}

// sweep_convert (scene.hpp:75): scene in, converted scene out (out's static
// arrays sized for n3 + n4), the moved dynamics indices and the report
int hgsr_sweep_convert(const hgso_scene* in, hgso_scene* out, int64_t* moved, hgso_conversion* rep) {
    try {
        hgs::HybridScene h = to_scene(*in);
        std::vector<std::size_t> mv;
        const hgs::ConversionReport r = hgs::sweep_convert(h, &mv);
        from_scene(h, *out);
        for (size_t i = 0; i < mv.size(); ++i) moved[i] = (int64_t)mv[i];
        rep->count = (int64_t)r.count;
        rep->max_leakage = r.max_leakage;
        rep->mean_leakage = r.mean_leakage;
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// optimizer_step (train.hpp:68-69) on fresh Adam state (step 0) with the
// given gradients: the updated scene (same sizes) and the skipped count
int hgsr_optimizer_step_fresh(const hgso_scene* in, const hgso_grads* g, const hgso_lrs* lrs, double mean_lr_scale,
                              int n_steps, hgso_scene* out, int64_t* skipped) {
    try {
        hgs::HybridScene h = to_scene(*in);
        const int K = hgs::sh_coeff_count(in->sh_degree);
        hgs::SceneGrads gr;
        gr.resize_like(h);
        for (int64_t i = 0; i < in->n4; ++i) {
            hgs::Grad4D& d = gr.dynamics[i];
            d.mean_x = hgs::Vec3(g->mean_x[3 * i], g->mean_x[3 * i + 1], g->mean_x[3 * i + 2]);
            d.mean_t = g->mean_t[i];
            d.quat_left = hgs::Vec4(g->ql[4 * i], g->ql[4 * i + 1], g->ql[4 * i + 2], g->ql[4 * i + 3]);
            d.quat_right = hgs::Vec4(g->qr[4 * i], g->qr[4 * i + 1], g->qr[4 * i + 2], g->qr[4 * i + 3]);
            d.log_scales = hgs::Vec4(g->log_s4[4 * i], g->log_s4[4 * i + 1], g->log_s4[4 * i + 2], g->log_s4[4 * i + 3]);
            d.opacity_logit = g->op4[i];
            for (int k = 0; k < K; ++k)
                d.sh[k] = hgs::Vec3(g->sh4[(i * K + k) * 3], g->sh4[(i * K + k) * 3 + 1], g->sh4[(i * K + k) * 3 + 2]);
        }
        for (int64_t i = 0; i < in->n3; ++i) {
            hgs::Grad3D& d = gr.statics[i];
            d.mean = hgs::Vec3(g->mean3[3 * i], g->mean3[3 * i + 1], g->mean3[3 * i + 2]);
            d.quat = hgs::Vec4(g->quat3[4 * i], g->quat3[4 * i + 1], g->quat3[4 * i + 2], g->quat3[4 * i + 3]);
            d.log_scales = hgs::Vec3(g->log_s3[3 * i], g->log_s3[3 * i + 1], g->log_s3[3 * i + 2]);
            d.opacity_logit = g->op3[i];
            for (int k = 0; k < K; ++k)
                d.sh[k] = hgs::Vec3(g->sh3[(i * K + k) * 3], g->sh3[(i * K + k) * 3 + 1], g->sh3[(i * K + k) * 3 + 2]);
        }
        hgs::GradAccum st;
        st.resize(h.statics.size(), h.dynamics.size(), 3 * (size_t)K);
        hgs::LearningRates l;
        l.mean = lrs->mean;
        l.mean_final_ratio = lrs->mean_final_ratio;
        l.mean_t = lrs->mean_t;
        l.quat = lrs->quat;
        l.scales = lrs->scales;
        l.opacity = lrs->opacity;
        l.sh = lrs->sh;
        for (int s = 0; s < n_steps; ++s) hgs::optimizer_step(h, gr, st, l, mean_lr_scale);
        from_scene(h, *out);
        *skipped = (int64_t)st.skipped_nonfinite;
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// save_checkpoint (data_io.hpp:91-92) of a scene and, when st != NULL, its
// GradAccum (m / v laid out like the scene arrays, optim.hpp:10-41)
int hgsr_save_checkpoint(const hgso_scene* s, double duration_seconds, const hgso_state* st, const char* path) {
    try {
        hgs::HybridScene h = to_scene(*s);
        h.duration_seconds = duration_seconds;
        const size_t n3 = (size_t)s->n3, n4 = (size_t)s->n4;
        const size_t K3 = 3 * (size_t)hgs::sh_coeff_count(s->sh_degree);
        hgs::GradAccum a;
        if (st) {
            a.resize(n3, n4, K3);
            auto cp = [](hgs::AdamBuf& b, const double* m, const double* v, size_t n) {
                b.m.assign(m, m + n);
                b.v.assign(v, v + n);
            };
            cp(a.statics.mean, st->m.mean3, st->v.mean3, 3 * n3);
            cp(a.statics.quat, st->m.quat3, st->v.quat3, 4 * n3);
            cp(a.statics.scales, st->m.log_s3, st->v.log_s3, 3 * n3);
            cp(a.statics.opacity, st->m.op3, st->v.op3, n3);
            cp(a.statics.sh, st->m.sh3, st->v.sh3, K3 * n3);
            cp(a.dynamics.mean_x, st->m.mean_x, st->v.mean_x, 3 * n4);
            cp(a.dynamics.mean_t, st->m.mean_t, st->v.mean_t, n4);
            cp(a.dynamics.quat_left, st->m.ql, st->v.ql, 4 * n4);
            cp(a.dynamics.quat_right, st->m.qr, st->v.qr, 4 * n4);
            cp(a.dynamics.scales, st->m.log_s4, st->v.log_s4, 4 * n4);
            cp(a.dynamics.opacity, st->m.op4, st->v.op4, n4);
            cp(a.dynamics.sh, st->m.sh4, st->v.sh4, K3 * n4);
            a.grad_norm3.assign(st->grad_norm3, st->grad_norm3 + n3);
            a.grad_norm4.assign(st->grad_norm4, st->grad_norm4 + n4);
            a.count3.assign(st->count3, st->count3 + n3);
            a.count4.assign(st->count4, st->count4 + n4);
            a.step = st->step;
            a.skipped_nonfinite = (size_t)st->skipped_nonfinite;
        }
        hgs::save_checkpoint(h, st ? &a : nullptr, path);
        return HGSO_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
