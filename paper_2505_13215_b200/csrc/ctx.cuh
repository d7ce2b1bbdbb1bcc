// ctx.cuh -- host-side context of the C ABI (one per GPU).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <string>
#include <vector>

#include "../../include/hgs_gpu.h"
#include "hgs_common.cuh"

namespace hgs {

struct DBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 2 + 4096;  // grow by 1.5x: steady state never reallocates
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct HostPinned {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes + bytes / 4 + 256;
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

// Buffers a render (and the training step around it) zeroes / fills before
// its kernels: one programmatic launch instead of a chain of memsets.
struct ZeroJob {
    void* p;
    uint64_t words;  // 32-bit words
    uint32_t value;
};
constexpr int kMaxZeroJobs = 10;
struct ZeroJobs {
    ZeroJob j[kMaxZeroJobs];
    int n = 0;
    void add(void* p, uint64_t bytes, uint32_t value = 0u) {
        if (!bytes) return;
        if (n >= kMaxZeroJobs) {  // a programming error: more fills than the launch carries
            fprintf(stderr, "hgs: ZeroJobs overflow\n");
            abort();
        }
        j[n++] = ZeroJob{p, bytes / 4, value};
    }
};

// Per-render device counters (RenderStats, flags, totals).
struct __align__(128) Counters {
    uint32_t flags;
    uint32_t V;
    uint32_t I;
    uint32_t fix_count;
    uint32_t skipped;
    uint32_t I_kept;
    uint32_t pad[26];
    unsigned long long stats[kStatStripes * kStatStride];  // striped RenderStats (K1)
    // RenderStats counter k summed over the stripes (host side)
    unsigned long long stat(int k) const {
        unsigned long long s = 0;
        for (int r = 0; r < kStatStripes; ++r) s += stats[r * kStatStride + k];
        return s;
    }
};

}  // namespace hgs

// One enqueued (pipelined) training iteration awaiting hgs_train_collect.
struct hgs_pending_step {
    int slot = 0, n_views = 0;
    int dims[32][2] = {};  // per view (W, H)
    double lambda = 0.2;
    bool adam = false;
    bool dist = false;  // completed by hgs_train_exchange_async (all-reduced abort decision)
    uint64_t step_before = 0;
};

struct hgs_ctx {
    bool stats_pending = false;  // counters of the last render not read back yet
    bool grads_zero = false;     // the packed gradient buffer is known to be all zero (K7/K7b store, no RMW)
    std::deque<hgs_pending_step> pipeline;  // hgs_train_step_async iterations, oldest first
    int pipe_next = 0;                      // next step-sum slot
    cudaEvent_t pipe_ev[HGS_TRAIN_PIPELINE] = {};
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    int sms = 148;

    // ---- device-resident scene (component-major SoA, see hgs_common.cuh)
    int64_t n4 = 0, n3 = 0, cap4 = 0, cap3 = 0;
    int deg = 1;
    double tau = 0.5, extent = 1.0, duration = 1.0;
    hgs::DBuf p4, p3;      // params
    hgs::DBuf p4_alt;      // compaction target of the 4D sweep
    hgs::DBuf m4_alt, v4_alt;
    // Packed gradient buffer (one contiguous allreduce payload):
    //   [g4: rows4*cap4 | g3: rows3*cap3 | dgn4: cap4 | dgn3: cap3 | dcnt4: cap4 | dcnt3: cap3]
    // g* share the parameter layout; d* are this step's densify-statistic
    // deltas (raw per-image screen norms and observation counts), folded into
    // gn/cnt by the Adam kernel.
    hgs::DBuf gbuf;
    float *g4 = nullptr, *g3 = nullptr, *dgn4 = nullptr, *dgn3 = nullptr, *dcnt4 = nullptr, *dcnt3 = nullptr;
    int64_t gbuf_floats = 0;
    hgs::DBuf m4, v4, m3, v3;  // Adam moments
    hgs::DBuf adam_ok;         // per-(class, Gaussian) finite flags (K8, 5 cap3 + 7 cap4 bytes)
    hgs::DBuf gn4, gn3;    // densify grad_norm (float)
    hgs::DBuf cnt4, cnt3;  // densify counts (float, exact below 2^24)
    hgs::DBuf sn4, sn3;    // screen_norm of the last backward (float)
    uint64_t step = 0;

    // ---- per-render workspace
    hgs::DBuf rec, depth_key, ntiles, visflag, vispos;
    hgs::DBuf sort_k, sort_v, sort_k2, sort_v2;       // depth sort (V)
    hgs::DBuf rec_sorted, fast_sorted, ntiles_sorted, inst_off, sorted_of_gid, pcut, dup_first;
    hgs::DBuf gpack;        // packed gradient payload (multi-GPU all-reduce)
    // densify_and_prune (densify.cu): plan buffers + planned sizes
    hgs::DBuf dens_cat, dens_u32, dens_misc, dens_kinds, dens_jit;
    bool dens_planned = false;
    int64_t dens_new[2] = {0, 0}, dens_count[2] = {0, 0};  // [statics, dynamics]
    hgs::DBuf dup_status;   // look-back status words of duplicate_compact_kernel
    hgs::DBuf shdir, ddir;  // K1 view direction + clamp mask; K7b dL/d(direction)
    hgs::DBuf inst_k, inst_v, inst_k2, inst_v2;       // tile sort (I)
    hgs::DBuf ranges, scan_ws, sort_ws, inst_flag, inst_pos;
    hgs::DBuf tile_order;  // the rasterizers' tile launch order (heaviest first; K4 and K6)
    hgs::DBuf dbg_k, dbg_v;         // the reference's full sorted instance list (debug / count_map)
    bool debug_full_list = false;   // hgs_debug_keep_instances
    bool skip_gid_map = false;  // render sweeps: a frame whose tape is not kept writes no gid -> sorted
                                // map and no depth-ordered SplatRec copy (K4 reads rec through the depth order)
    hgs::DBuf counters;  // [0..5] stats u64, [6] flags, fix_count, totals...
    hgs::DBuf img, last, tfinal, trans, count, fix_list;
    hgs::DBuf fix_cout;  // FP64 colours of the fix-up pixels (forward fix-up -> exact backward)
    hgs::DBuf fix_slot;  // per pixel: its fix-list slot (written for the fix-up pixels only)
    hgs::DBuf accum;     // backward per-sorted-splat accumulators
    bool exact_backward = false;  // hgs_set_exact_backward: FP64 pair terms for every pixel
    hgs::DBuf exact_col;          // its FP64 colours (sorted order)
    hgs::DBuf lgrad;     // dL/dimage (device float)
    hgs::DBuf loss_img;  // the image of a standalone hgs_photometric_loss_with_grad
    hgs::DBuf gt_stage;  // staged ground truth
    hgs::DBuf gt_buf[2], gt_stage64[2];  // double-buffered host GT of the training step
    cudaStream_t copy_stream = nullptr;  // host -> device GT copies, overlapped with the render
    cudaEvent_t gt_ready[2] = {nullptr, nullptr}, gt_free[2] = {nullptr, nullptr};
    hgs::DBuf loss_ws;   // loss scratch (SSIM maps)
    hgs::DBuf scratch;   // small device scalars (loss sums, skip counts, leakage)
    hgs::DBuf stage;     // upload / download staging
    hgs::DBuf dmap;      // density_map difference array ((W+1)*(H+1) ints) and counts
    hgs::DBuf ckpt;              // checkpoint payloads on the device (checkpoint.cu)
    hgs::DBuf crc_tab;           // CRC-32 slicing tables (checkpoint.cu)
    void* comm = nullptr;        // ncclComm_t of the view-parallel exchange (comm.cu)
    int comm_rank = 0, comm_size = 1;
    bool sharded = false;      // hgs_comm_set_sharded: reduce-scatter / sharded Adam / all-gather
    bool state_sharded = false;  // Adam moments valid only on this rank's shard (hgs_gather_state)
    hgs::DBuf comm_buf;          // small staging for collectives / checksums
    uint32_t icap = 0;           // instance capacity of capacity-mode renders (hgs_render_sweep)
    int64_t redone_frames = 0;   // sweep frames re-rendered after a capacity overflow
    hgs::DBuf sweep_ctr;         // per-frame Counters of a sweep
    hgs::HostPinned sweep_host;
    hgs::HostPinned ckpt_host;   // checkpoint file image
    hgs::HostPinned pinned;      // Scratch read-back (training / loss)
    hgs::HostPinned pinned_ctr;  // Counters read-back (render)
    hgs::HostPinned pinned_pipe; // per-slot loss sums of pipelined iterations

    // ---- state of the last render (the "tape")
    bool have_tape = false;
    int W = 0, H = 0, tiles_x = 0, tiles_y = 0;
    int64_t V = 0, I = 0;
    uint32_t* inst_vals_final = nullptr;  // tile-sorted instance values the rasterizers walk (culled)
    uint32_t* inst_keys_all = nullptr;    // full tile-sorted instance list (reference semantics)
    uint32_t* inst_vals_all = nullptr;
    int64_t kept = 0;
    hgs::DevCamera cam{};
    double t = 0.0;
    double bg[3] = {0, 0, 0};
    int64_t fixups = 0, fp64_splats = 0;
    hgs_render_stats stats{};
    uint32_t* sorted_gid = nullptr;       // V sorted gids

    // ---- optional per-phase CUDA-event timing (bench.py roofline)
    bool profile = false;
    struct ProfEvent {
        int phase;
        cudaEvent_t a, b;
    };
    std::vector<cudaEvent_t> ev_pool;
    std::vector<ProfEvent> ev_pending;
    double phase_ms[16] = {0};
    long long phase_calls[16] = {0};
};

// Phases timed by the profiler (hgs_profile_read order).
enum HgsPhase {
    PH_PREPROCESS = 0,  // K1 + visibility compaction
    PH_DEPTH_SORT = 1,  // stable radix sort by f32 depth
    PH_DUPLICATE = 2,   // gather + tile-count scan + K2 duplication
    PH_TILE_SORT = 3,   // stable radix sort by tile + ranges
    PH_RASTER_FWD = 4,  // K4 + FP64 fix-up
    PH_LOSS = 5,        // K5
    PH_RASTER_BWD = 6,  // K6 + exact pixels
    PH_GAUSS_BWD = 7,   // K7
    PH_ADAM = 8,        // K8 + statistic fold
    PH_SWEEP = 9,       // K9
    PH_UPLOAD = 10,     // host->device copies of the e2e path
};

void prof_begin(hgs_ctx* ctx, int phase);
void prof_end(hgs_ctx* ctx);
void prof_collect(hgs_ctx* ctx);
