// rng.cpp -- the training loop's random stream (train.cpp:68-72, 245-275,
// 387-404) as a C-ABI object, so a C++ caller (and the Python driver) get
// the reference's batch schedule and densification jitter bit for bit: the
// same libstdc++ std::mt19937_64, std::uniform_int_distribution<size_t> and
// std::normal_distribution<double> the reference instantiates, drawn in the
// reference's order.  Only the few draws of a densification run on the host;
// everything they feed is applied on the device (densify.cu).
#include <algorithm>
#include <cstdint>
#include <new>
#include <random>
#include <vector>

#include "../../include/hgs_gpu.h"

struct hgs_rng {
    std::mt19937_64 eng;
};

extern "C" {

hgs_status hgs_rng_create(uint64_t seed, hgs_rng** out) {
    if (!out) return HGS_ERR_INVALID_ARGUMENT;
    *out = new (std::nothrow) hgs_rng{std::mt19937_64(seed)};
    return *out ? HGS_OK : HGS_ERR_INVALID_ARGUMENT;
}

void hgs_rng_destroy(hgs_rng* r) { delete r; }

uint64_t hgs_rng_raw(hgs_rng* r) { return r ? r->eng() : 0; }

uint64_t hgs_rng_index(hgs_rng* r, uint64_t lo, uint64_t hi) {
    if (!r || hi < lo) return lo;
    std::uniform_int_distribution<std::size_t> d(lo, hi);
    return d(r->eng);
}

// train.cpp:403-404: `count` picks of samples[pick(rng)], pick over [0, n-1]
hgs_status hgs_rng_batch(hgs_rng* r, uint64_t n_samples, int32_t count, uint64_t* out) {
    if (!r || !out || n_samples == 0 || count < 0) return HGS_ERR_INVALID_ARGUMENT;
    std::uniform_int_distribution<std::size_t> pick(0, n_samples - 1);
    for (int32_t i = 0; i < count; ++i) out[i] = pick(r->eng);
    return HGS_OK;
}

// The normals densify_and_prune draws, laid out for hgs_densify_apply.
// Statics (train.cpp:68-72, 207-235): a fresh distribution per
// sample_normal3, a, b, c drawn in order; 6 doubles per densified Gaussian
// (clone: one triple; split: two).  Dynamics (train.cpp:245-275): ONE
// distribution for the pool; Vec4 n(nd(rng), nd(rng), nd(rng), nd(rng)) --
// g++ evaluates the four arguments right to left, so the first draw is the
// last component; 8 doubles per densified Gaussian.
hgs_status hgs_densify_normals(hgs_rng* r, const uint8_t* kinds3, int64_t d3, const uint8_t* kinds4, int64_t d4,
                               double* normals3, double* normals4) {
    if (!r || d3 < 0 || d4 < 0 || (d3 && (!kinds3 || !normals3)) || (d4 && (!kinds4 || !normals4)))
        return HGS_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < d3; ++i)
        for (int h = 0; h < (kinds3[i] == 1 ? 1 : 2); ++h) {
            std::normal_distribution<double> nd(0.0, 1.0);
            const double a = nd(r->eng), b = nd(r->eng), c = nd(r->eng);
            double* o = normals3 + 6 * i + 3 * h;
            o[0] = a;
            o[1] = b;
            o[2] = c;
        }
    std::normal_distribution<double> nd(0.0, 1.0);
    for (int64_t i = 0; i < d4; ++i)
        for (int h = 0; h < (kinds4[i] == 1 ? 1 : 2); ++h) {
            const double first = nd(r->eng), second = nd(r->eng), third = nd(r->eng), fourth = nd(r->eng);
            double* o = normals4 + 8 * i + 4 * h;
            o[0] = fourth;
            o[1] = third;
            o[2] = second;
            o[3] = first;
        }
    return HGS_OK;
}

// densify_and_prune (train.cpp:182-299) in one call: plan on the device,
// the jitter draws here, apply on the device.
hgs_status hgs_densify_and_prune(hgs_ctx* ctx, const hgs_densify_cfg* cfg, hgs_rng* r, hgs_densify_report* report) {
    if (!ctx || !cfg || !r) return HGS_ERR_INVALID_ARGUMENT;
    int64_t n4 = 0, n3 = 0;
    int32_t deg = 0;
    hgs_status s = hgs_scene_counts(ctx, &n4, &n3, &deg);
    if (s != HGS_OK) return s;
    std::vector<uint8_t> k3((size_t)std::max<int64_t>(n3, 1)), k4((size_t)std::max<int64_t>(n4, 1));
    hgs_densify_report rep{};
    s = hgs_densify_plan(ctx, cfg, k3.data(), k4.data(), &rep);
    if (s != HGS_OK) return s;
    const int64_t d3 = rep.cloned3 + rep.split3, d4 = rep.cloned4 + rep.split4;
    std::vector<double> nr3((size_t)std::max<int64_t>(6 * d3, 1)), nr4((size_t)std::max<int64_t>(8 * d4, 1));
    s = hgs_densify_normals(r, k3.data(), d3, k4.data(), d4, nr3.data(), nr4.data());
    if (s != HGS_OK) return s;
    s = hgs_densify_apply(ctx, nr3.data(), nr4.data(), cfg->split_factor);
    if (s == HGS_OK && report) *report = rep;
    return s;
}

}  // extern "C"
