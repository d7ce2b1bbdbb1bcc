// train_api.cuh -- host-side entry points shared between capi.cu and train.cu
#pragma once
#include "ctx.cuh"

// deferred != 0: leave the final counter read-back (stats, flags) to
// hgs_render_finish (the training step does it once at its end)
// icap > 0: capacity mode (no host round trip, see capi.cu); counters_slot:
// a device Counters record to use instead of the context's
// extra: buffers to fill in the render's own fill launch (training step)
hgs_status hgs_render_pipeline(hgs_ctx* ctx, const hgs_camera* cam, double t, const double bg[3],
                               const hgs_raster_opts* opts, int deferred = 0, uint32_t icap = 0,
                               void* counters_slot = nullptr, const hgs::ZeroJobs* extra = nullptr);
hgs_status hgs_render_finish(hgs_ctx* ctx);
hgs_status hgs_upload_rows(hgs_ctx* ctx, const hgs_host_scene* s, int dtype, float* dst4, float* dst3);
hgs_status hgs_layout_state(hgs_ctx* ctx);
// GradAccum::skipped_nonfinite on the device: read (get) and / or overwrite (set)
hgs_status hgs_skipped_total(hgs_ctx* ctx, uint64_t* get, const uint64_t* set);
// (Re)allocates the device pools for n4 / n3 Gaussians of degree deg, zeroes
// the optimizer state and statistics (the allocation half of hgs_scene_upload)
hgs_status hgs_scene_alloc(hgs_ctx* ctx, int64_t n4, int64_t n3, int deg, double tau, double extent,
                           double duration);
// stream-ordered all-reduce (sum) of n device doubles over the context's communicator (comm.cu)
hgs_status comm_allreduce_f64_dev(hgs_ctx* ctx, double* dev, int n);
// sharded optimizer exchange (comm.cu, hgs_comm_set_sharded)
hgs_status comm_reduce_scatter_grads(hgs_ctx* ctx);
hgs_status comm_sharded_finish(hgs_ctx* ctx, unsigned long long* skipped, unsigned long long* skipped_cum);
