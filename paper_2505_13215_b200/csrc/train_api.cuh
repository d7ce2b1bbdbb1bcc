// train_api.cuh -- host-side entry points shared between capi.cu and train.cu
#pragma once
#include "ctx.cuh"

// deferred != 0: leave the final counter read-back (stats, flags) to
// hgs_render_finish (the training step does it once at its end)
hgs_status hgs_render_pipeline(hgs_ctx* ctx, const hgs_camera* cam, double t, const double bg[3],
                               const hgs_raster_opts* opts, int deferred = 0);
hgs_status hgs_render_finish(hgs_ctx* ctx);
hgs_status hgs_upload_rows(hgs_ctx* ctx, const hgs_host_scene* s, int dtype, float* dst4, float* dst3);
hgs_status hgs_layout_state(hgs_ctx* ctx);
