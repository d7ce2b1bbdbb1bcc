// backend_demo.cpp -- a C++ program written against the REFERENCE's own API
// (/root/reference/proj/include/hgs) that calls the reference's CPU
// implementation (hgs::...) and the B200 backend with the same signatures
// (hgs::gpu::..., paper_2505_13215_b200/host/gpu_backend.hpp) side by side on
// the reference's own synthetic benchmark (generate_synthetic, data_io.cpp),
// and prints one JSON line per check for tests/test_gpu_cpp_backend.py.
//
// Built by examples/Makefile (needs the reference headers and objects:
// oracle/_ref); the binary travels to the GPU box prebuilt.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "gpu_backend.hpp"
#include "hgs/data_io.hpp"
#include "hgs/metrics.hpp"

using namespace hgs;

static double max_abs_diff(const std::vector<double>& a, const std::vector<double>& b) {
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

static bool same_stats(const RenderStats& a, const RenderStats& b) {
    return a.culled_depth == b.culled_depth && a.culled_offscreen == b.culled_offscreen &&
           a.culled_degenerate == b.culled_degenerate && a.culled_temporal == b.culled_temporal &&
           a.degenerate_temporal == b.degenerate_temporal && a.projected == b.projected;
}

// Flattened gradients (every class, both pools) for a norm-wise comparison,
// plus the per-element relative error with the 1e-6 floor.
static std::vector<double> flat(const SceneGrads& g) {
    std::vector<double> v;
    for (const auto& d : g.dynamics) {
        for (int k = 0; k < 3; ++k) v.push_back(d.mean_x[k]);
        v.push_back(d.mean_t);
        for (int k = 0; k < 4; ++k) v.push_back(d.quat_left[k]);
        for (int k = 0; k < 4; ++k) v.push_back(d.quat_right[k]);
        for (int k = 0; k < 4; ++k) v.push_back(d.log_scales[k]);
        v.push_back(d.opacity_logit);
        for (const Vec3& c : d.sh)
            for (int k = 0; k < 3; ++k) v.push_back(c[k]);
    }
    for (const auto& d : g.statics) {
        for (int k = 0; k < 3; ++k) v.push_back(d.mean[k]);
        for (int k = 0; k < 4; ++k) v.push_back(d.quat[k]);
        for (int k = 0; k < 3; ++k) v.push_back(d.log_scales[k]);
        v.push_back(d.opacity_logit);
        for (const Vec3& c : d.sh)
            for (int k = 0; k < 3; ++k) v.push_back(c[k]);
    }
    return v;
}

static std::vector<double> flat(const HybridScene& s) {
    std::vector<double> v;
    for (const auto& g : s.dynamics) {
        for (int k = 0; k < 3; ++k) v.push_back(g.mean_x[k]);
        v.push_back(g.mean_t);
        for (double q : {g.rot.left.w, g.rot.left.x, g.rot.left.y, g.rot.left.z, g.rot.right.w, g.rot.right.x,
                         g.rot.right.y, g.rot.right.z})
            v.push_back(q);
        for (int k = 0; k < 4; ++k) v.push_back(g.log_scales[k]);
        v.push_back(g.opacity_logit);
        for (const Vec3& c : g.color.coeffs)
            for (int k = 0; k < 3; ++k) v.push_back(c[k]);
    }
    for (const auto& g : s.statics) {
        for (int k = 0; k < 3; ++k) v.push_back(g.mean[k]);
        for (double q : {g.rot.w, g.rot.x, g.rot.y, g.rot.z}) v.push_back(q);
        for (int k = 0; k < 3; ++k) v.push_back(g.log_scales[k]);
        v.push_back(g.opacity_logit);
        for (const Vec3& c : g.color.coeffs)
            for (int k = 0; k < 3; ++k) v.push_back(c[k]);
    }
    return v;
}

int main() {
    std::setvbuf(stdout, nullptr, _IOLBF, 0);
    SynthSpec spec;  // the reference's defaults: 60 static + 3 x 8 dynamic, 4 cameras x 20 frames, 64x64
    const SyntheticScene syn = generate_synthetic(spec, 7);
    const MultiViewDataset& ds = syn.dataset;
    const HybridScene& gt = syn.ground_truth;
    const Camera& cam = ds.cameras[1];
    const double t = ds.frames[1][7].time;

    // 1. rasterize (raster.hpp:79-80)
    RasterOpts ro;
    ro.count_map = ro.transmittance_map = true;
    const RenderOutput a = rasterize(gt, cam, t, ds.background, ro);
    const RenderOutput b = gpu::rasterize(gt, cam, t, ds.background, ro);
    std::printf("{\"check\": \"rasterize\", \"max_abs\": %.3e, \"counts_equal\": %d, \"trans_max_abs\": %.3e, "
                "\"stats_equal\": %d, \"projected\": %zu}\n",
                max_abs_diff(a.rgb.data, b.rgb.data), a.counts == b.counts ? 1 : 0,
                max_abs_diff(a.transmittance, b.transmittance), same_stats(a.stats, b.stats) ? 1 : 0,
                b.stats.projected);

    // 2. forward_train + photometric_loss_with_grad + backward (backward.hpp:68-74)
    InitConfig ic;
    ic.sh_degree = 1;
    ic.duration_seconds = ds.duration_seconds;
    const HybridScene init = init_scene(syn.init_points, ic);
    const Frame& fr = ds.frames[2][5];
    Tape ta, tb;
    const Image ia = forward_train(init, ds.cameras[2], fr.time, ds.background, {}, ta);
    const Image ib = gpu::forward_train(init, ds.cameras[2], fr.time, ds.background, {}, tb);
    Image la, lb;
    const double loss_a = photometric_loss_with_grad(ia, fr.image, 0.2, la);
    const double loss_b = gpu::photometric_loss_with_grad(ib, fr.image, 0.2, lb);
    SceneGrads ga, gb;
    ga.resize_like(init);
    gb.resize_like(init);
    backward(init, ds.cameras[2], ta, la, ga);
    gpu::backward(init, ds.cameras[2], tb, la, gb);  // the same dL/dimage on both sides
    const std::vector<double> fa = flat(ga), fb = flat(gb);
    double na = 0, nd = 0, worst = 0;
    size_t bad = 0;
    for (size_t i = 0; i < fa.size(); ++i) {
        na += fa[i] * fa[i];
        nd += (fa[i] - fb[i]) * (fa[i] - fb[i]);
        const double r = std::abs(fa[i] - fb[i]) / std::max({std::abs(fa[i]), std::abs(fb[i]), 1e-6});
        worst = std::max(worst, r);
        bad += r > 1e-3;
    }
    std::printf("{\"check\": \"forward_backward\", \"image_max_abs\": %.3e, \"loss_ref\": %.12g, \"loss_gpu\": %.12g, "
                "\"grad_rel_norm\": %.3e, \"grad_max_rel\": %.3e, \"grad_n_bad\": %zu, \"n\": %zu}\n",
                max_abs_diff(ia.data, ib.data), loss_a, loss_b, std::sqrt(nd / std::max(na, 1e-300)), worst, bad,
                fa.size());

    // 3. optimizer_step (train.hpp:68-69) on the same gradients, 3 steps
    HybridScene sa = init, sb = init;
    GradAccum sta, stb;
    sta.resize(sa.statics.size(), sa.dynamics.size(), 3 * (size_t)sh_coeff_count(sa.sh_degree));
    stb = sta;
    LearningRates lr;
    for (int k = 0; k < 3; ++k) {
        optimizer_step(sa, ga, sta, lr, 0.8);
        gpu::optimizer_step(sb, ga, stb, lr, 0.8);
    }
    std::printf("{\"check\": \"optimizer_step\", \"param_max_abs\": %.3e, \"step_ref\": %llu, \"step_gpu\": %llu, "
                "\"m_max_abs\": %.3e}\n",
                max_abs_diff(flat(sa), flat(sb)), (unsigned long long)sta.step, (unsigned long long)stb.step,
                max_abs_diff(sta.dynamics.mean_x.m, stb.dynamics.mean_x.m));

    // 5. train (train.hpp:88): the reference's loop on the CPU and the
    //    device-resident loop, same dataset / config / seed
    TrainConfig cfg;
    cfg.iterations = 40;
    cfg.batch_size = 2;
    cfg.warmup_iters = 10;
    cfg.densify_interval = 10;
    cfg.densify_stop_iter = 30;
    cfg.probe_interval = 10;
    cfg.seed = 3;
    cfg.num_threads = 2;
    cfg.tau = 0.105;  // init_temporal_scale 0.1: the sweeps convert the Gaussians whose s_t grew
    const TrainResult ta_ = train(ds, cfg);
    const TrainResult tb_ = gpu::train(ds, cfg);
    std::printf("{\"check\": \"train\", \"rows\": %zu, \"loss1_ref\": %.9g, \"loss1_gpu\": %.9g, "
                "\"psnr_ref\": %.6g, \"psnr_gpu\": %.6g, \"n_ref\": [%zu, %zu], \"n_gpu\": [%zu, %zu], "
                "\"conv_ref\": %zu, \"conv_gpu\": %zu, \"step_gpu\": %llu}\n",
                tb_.log.rows.size(), ta_.log.rows.front().loss, tb_.log.rows.front().loss,
                ta_.log.rows.back().probe_psnr, tb_.log.rows.back().probe_psnr, ta_.scene.statics.size(),
                ta_.scene.dynamics.size(), tb_.scene.statics.size(), tb_.scene.dynamics.size(),
                ta_.log.rows[9].conversions + ta_.log.rows[19].conversions,
                tb_.log.rows[9].conversions + tb_.log.rows[19].conversions, (unsigned long long)tb_.state.step);

    // 6. sweep_convert (scene.hpp:75) on the reference-trained scene
    HybridScene ca = ta_.scene, cb = ta_.scene;
    ca.tau = cb.tau = 0.1;
    std::vector<size_t> ma, mb;
    const ConversionReport ra = sweep_convert(ca, &ma);
    const ConversionReport rb = gpu::sweep_convert(cb, &mb);
    std::printf("{\"check\": \"sweep_convert\", \"count_ref\": %zu, \"count_gpu\": %zu, \"moved_equal\": %d, "
                "\"pool_max_abs\": %.3e, \"leak_ref\": %.12g, \"leak_gpu\": %.12g}\n",
                ra.count, rb.count, ma == mb ? 1 : 0, max_abs_diff(flat(ca), flat(cb)), ra.max_leakage,
                rb.max_leakage);

    // 7. the reference's exception types through the boundary
    int typed = 0;
    try {
        Camera bad = cam;
        bad.fx = -1;
        gpu::rasterize(gt, bad, t, ds.background);
    } catch (const std::invalid_argument&) {
        typed = 1;
    }
    std::printf("{\"check\": \"errors\", \"invalid_argument\": %d}\n", typed);
    return 0;
}
