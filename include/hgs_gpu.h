/*
 * hgs_gpu.h -- C ABI of the B200-native (sm_100a) hybrid 3D/4DGS hot path.
 *
 * This is the drop-in boundary: plain pointers, sizes and POD structs, no
 * torch or CUDA types.  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj).  INTEGRATION.md shows
 * the C++ shim (hgs::rasterize etc. over this ABI) and the pybind / ctypes
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *   - One hgs_ctx per GPU, used by one host thread.  Calls are
 *     stream-ordered on the context's stream; the "host" entry points
 *     (hgs_rasterize, hgs_render with host outputs) synchronise before
 *     returning, the device-resident training entry points do not.
 *   - Every function returns an hgs_status; on error hgs_last_error(ctx)
 *     holds a message.  The C++ shim maps statuses back to the reference's
 *     exception types (errors.hpp:9-33 / std::invalid_argument).
 *   - There is no CPU fallback: without a usable CUDA device every call that
 *     needs one returns HGS_ERR_CUDA.
 *   - Scene buffers follow the reference's per-class layout (scene.hpp:13-59):
 *     row-major per Gaussian, quaternions (w,x,y,z), SH as K=(deg+1)^2 RGB
 *     triples.  dtype selects double (HGS_F64, the reference's precision) or
 *     float (HGS_F32) host arrays.  On the device parameters are FP32 SoA.
 */
#ifndef HGS_GPU_H
#define HGS_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HGS_OK = 0,
    HGS_ERR_INVALID_ARGUMENT = 1,    /* std::invalid_argument */
    HGS_ERR_DEGENERATE_TEMPORAL = 2, /* DegenerateTemporalError */
    HGS_ERR_DEGENERATE_ROTATION = 3, /* DegenerateRotationError */
    HGS_ERR_NUMERIC_ABORT = 4,       /* NumericAbort */
    HGS_ERR_CUDA = 5,                /* no device / launch failure */
    HGS_ERR_STATE = 6,               /* call out of order (e.g. backward before forward) */
    HGS_ERR_FORMAT = 7,              /* FormatError (checkpoint / dataset files) */
    HGS_ERR_INTEGRITY = 8,           /* IntegrityError (checkpoint checksum) */
    HGS_ERR_UNSUPPORTED_VERSION = 9  /* UnsupportedVersionError */
} hgs_status;

enum { HGS_F64 = 0, HGS_F32 = 1, HGS_U8 = 2 };
/* HGS_U8: ground-truth frames only -- 8-bit sRGB RGB triples as the dataset
 * stores them (read_ppm), decoded on the device with srgb8_to_linear
 * (image.cpp:20-22, (v/255)^2.2) inside the loss: 4x less memory and
 * host->device traffic than float frames, identical loss values. */

typedef struct hgs_ctx hgs_ctx;

/* Host view of a HybridScene (scene.hpp:49-59).  Pointers are double* or
 * float* according to the dtype argument of the call that takes it. */
typedef struct {
    int64_t n4, n3;
    int32_t sh_degree;
    double tau, extent;
    void *mean_x, *mean_t, *ql, *qr, *log_s4, *op4, *sh4; /* dynamics */
    void *mean3, *quat3, *log_s3, *op3, *sh3;             /* statics  */
    double duration_seconds;                              /* scene.hpp:52 */
} hgs_host_scene;

/* Host view of the optimizer state GradAccum (optim.hpp:32-41): Adam
 * moments laid out like the scene (only the pointer fields of m / v are
 * read), densification statistics, step and skipped-row counters.
 * Always double / uint32 (HGS_F64). */
typedef struct {
    uint64_t step, skipped_nonfinite;
    hgs_host_scene m, v;
    double *grad_norm4, *grad_norm3;
    uint32_t *count4, *count3;
} hgs_host_state;

/* Camera (camera.hpp:11-16): x_cam = rot * x + trans, rot row-major. */
typedef struct {
    double fx, fy, cx, cy;
    double rot[9];
    double trans[3];
    int32_t width, height;
    double near_, far_;
} hgs_camera;

/* RenderStats (raster.hpp:33-40), counts identical to the reference. */
typedef struct {
    int64_t culled_depth, culled_offscreen, culled_degenerate, culled_temporal,
        degenerate_temporal, projected;
} hgs_render_stats;

/* RasterOpts (raster.hpp:42-47); num_threads is accepted and ignored (the
 * CUDA grid replaces the tile thread pool; output is thread-count invariant
 * exactly as in the reference). */
typedef struct {
    double weight_cutoff;
    int32_t num_threads;
    int32_t count_map;
    int32_t transmittance_map;
} hgs_raster_opts;

/* LearningRates (train.hpp:13-21) */
typedef struct {
    double mean, mean_final_ratio, mean_t, quat, scales, opacity, sh;
} hgs_lrs;

/* ConversionReport (scene.hpp:38-42) */
typedef struct {
    int64_t count;
    double max_leakage, mean_leakage;
} hgs_conversion_report;

/* Per-render diagnostics (not in the reference): visible splats, tile
 * instances (the reference's list), instances the rasterizers walk after the
 * exact tile-ellipse culling, and pixels recomposited by the FP64 fix-up. */
typedef struct {
    int64_t visible, instances, fixup_pixels, kept_instances;
    int64_t sweep_redone_frames; /* hgs_render_sweep frames re-rendered after a capacity overflow (total) */
} hgs_render_info;

/* ---- lifecycle -------------------------------------------------------- */
hgs_status hgs_ctx_create(int device, hgs_ctx **out);
void hgs_ctx_destroy(hgs_ctx *ctx);
const char *hgs_last_error(const hgs_ctx *ctx);
/* cudaStream_t as void*; NULL = the context's own stream */
hgs_status hgs_ctx_set_stream(hgs_ctx *ctx, void *stream);
void *hgs_ctx_stream(hgs_ctx *ctx);
hgs_status hgs_synchronize(hgs_ctx *ctx);

/* ---- scene (device resident) ------------------------------------------ */
/* Upload a host scene; resets the optimizer state and gradients. */
hgs_status hgs_scene_upload(hgs_ctx *ctx, const hgs_host_scene *scene, int dtype);
/* Download into caller buffers sized for hgs_scene_counts(). */
hgs_status hgs_scene_download(hgs_ctx *ctx, hgs_host_scene *out, int dtype);
hgs_status hgs_scene_counts(hgs_ctx *ctx, int64_t *n4, int64_t *n3, int32_t *sh_degree);

/* ---- rendering: rasterize (raster.hpp:79-80) --------------------------- */
/* Literal drop-in: uploads `scene`, renders, downloads.  rgb_out is an
 * (h, w, 3) array of dtype; counts/trans are optional (h, w) maps. */
hgs_status hgs_rasterize(hgs_ctx *ctx, const hgs_host_scene *scene, int dtype, const hgs_camera *cam,
                         double t, const double bg[3], const hgs_raster_opts *opts, void *rgb_out,
                         uint32_t *count_out, void *trans_out, hgs_render_stats *stats);
/* Render the device-resident scene.  Host outputs (any may be NULL). */
hgs_status hgs_render(hgs_ctx *ctx, const hgs_camera *cam, double t, const double bg[3],
                      const hgs_raster_opts *opts, float *rgb_host, uint32_t *count_host,
                      float *trans_host, hgs_render_stats *stats);
/* Render sweep (config c5): n frames (cams[f], ts[f]) of the resident scene
 * with no host round trip between them and one synchronisation at the end;
 * out (optional; n * h * w * 3 floats, all cameras the same size) is a
 * device pointer when out_on_device, else host memory; stats (optional) has
 * n entries.  Identical images to n hgs_render calls: the instance buffers
 * are sized from a capacity learned on the context, and a frame that
 * exceeded it is re-rendered exactly before the call returns. */
hgs_status hgs_render_sweep(hgs_ctx *ctx, int n, const hgs_camera *cams, const double *ts, const double bg[3],
                            const hgs_raster_opts *opts, float *out, int out_on_device,
                            hgs_render_stats *stats);
/* Device pointer of the last rendered image (float, h*w*3), valid until the
 * next render on this context. */
const float *hgs_last_image_device(hgs_ctx *ctx);
hgs_status hgs_render_info_get(hgs_ctx *ctx, hgs_render_info *info);

/* ---- differentiable forward / backward (backward.hpp:68-74) ------------ */
/* forward_train: renders and keeps the (opaque, device) tape. */
hgs_status hgs_forward_train(hgs_ctx *ctx, const hgs_camera *cam, double t, const double bg[3],
                             const hgs_raster_opts *opts, float *rgb_host);
/* backward: dL/dimage (h*w*3, host dtype or device float when on_device),
 * accumulated as scale * grad into the context's gradient buffer; also
 * updates the densification statistics (train.cpp:433-444) with the raw
 * per-image screen-space norms. */
hgs_status hgs_backward(hgs_ctx *ctx, const void *loss_grad, int dtype, int on_device, double scale);
/* Exact backward mode (default off): every pixel's pair terms in FP64 with
 * FP64 colours, the reference's own arithmetic (backward.cpp:178-356), at
 * several times the cost of the default path -- whose FP32 pair terms
 * (FP64 accumulation) meet the 1e-3 per-element gate at the training
 * configurations but not for adversarial, strongly cancelling loss
 * gradients. */
hgs_status hgs_set_exact_backward(hgs_ctx *ctx, int enable);
hgs_status hgs_zero_grads(hgs_ctx *ctx);
/* Download gradients in the scene layout (double or float), plus the
 * screen_norm of the LAST backward call (backward.hpp:20, 30). */
hgs_status hgs_grads_download(hgs_ctx *ctx, hgs_host_scene *out, int dtype, void *screen_norm4,
                              void *screen_norm3);
/* Packed device gradient buffer (for the view-parallel allreduce). */
hgs_status hgs_grads_device(hgs_ctx *ctx, float **ptr, int64_t *count);
/* Packed gradient payload for a multi-GPU all-reduce: unpack = 0 fills a
 * context-owned device buffer with the valid part of every gradient row and
 * the densify-statistic deltas (ptr/count out); unpack = 1 scatters that
 * buffer (reduced in place by the caller, e.g. ncclAllReduce) back. */
hgs_status hgs_grads_packed(hgs_ctx *ctx, int unpack, float **ptr, int64_t *count);

/* ---- multi-GPU exchange -------------------------------- */
/* View-parallel data parallelism: each rank renders its views with
 * apply_adam = 0, hgs_allreduce_grads sums the gradient rows + the
 * densify-statistic deltas over the ranks in place (one NCCL group of
 * all-reduces over the valid prefix of every row, on the context stream; no
 * packing), then every rank runs the same hgs_adam_step.  NCCL is
 * loaded at run time (libnccl.so.2; an already-loaded copy is shared).
 *   hgs_comm_unique_id  -- on one rank; ship the 128 bytes out of band
 *   hgs_comm_init       -- one process per GPU (ncclCommInitRank)
 *   hgs_comm_init_all   -- one process driving n contexts (ncclCommInitAll)
 *   hgs_allreduce_f64   -- sum of n host doubles over the ranks (the batch
 *                          loss: every rank raises NumericAbort together)
 *   hgs_param_checksum  -- order-independent 64-bit checksum of the
 *                          parameters (replica-consistency check)
 *   hgs_broadcast_params -- parameters, Adam moments and statistics from
 *                          `root` (repairs diverged replicas) */
typedef struct {
    char internal[128];
} hgs_comm_id;
hgs_status hgs_comm_unique_id(hgs_comm_id *out);
hgs_status hgs_comm_init(hgs_ctx *ctx, int nranks, int rank, const hgs_comm_id *id);
hgs_status hgs_comm_init_all(hgs_ctx *const *ctxs, int n);
hgs_status hgs_comm_destroy(hgs_ctx *ctx);
/* The NCCL the exchange binds (the copy already mapped into the process --
 * e.g. torch's -- else libnccl.so.2): version code and library path. */
hgs_status hgs_comm_nccl_info(int *version, char *path, int path_len);
int hgs_comm_size(hgs_ctx *ctx);
int hgs_comm_rank(hgs_ctx *ctx);
hgs_status hgs_allreduce_grads(hgs_ctx *ctx);
hgs_status hgs_allreduce_f64(hgs_ctx *ctx, double *vals, int n);
hgs_status hgs_param_checksum(hgs_ctx *ctx, uint64_t *out);
hgs_status hgs_broadcast_params(hgs_ctx *ctx, int root);

/* ---- loss (loss.hpp:12-13) --------------------------------------------- */
/* (1-l)*L1 + l*(1-SSIM) of the last rendered image against gt (h*w*3, host
 * dtype or device float); dL/dimage stays on the device for hgs_backward. */
hgs_status hgs_loss_with_grad(hgs_ctx *ctx, const void *gt, int dtype, int on_device, double ssim_lambda,
                              double *loss_out, void *grad_host_out);
/* Standalone: loss and gradient of two host images. */
hgs_status hgs_photometric_loss_with_grad(hgs_ctx *ctx, const void *rendered, const void *gt, int dtype,
                                          int width, int height, double ssim_lambda, double *loss_out,
                                          void *grad_out);

/* ---- evaluation (eval.cpp:12-23, metrics.cpp:91-101, raster.cpp:268-287) */
/* PSNR (peak 1) and mean SSIM (valid 11x11 windows, over channels) of the
 * last rendered image against gt (h*w*3: host HGS_F64/HGS_F32/HGS_U8, or a
 * device HGS_F32/HGS_U8 frame when on_device).  psnr is +inf for identical
 * images; asking for ssim of an image smaller than the window is
 * HGS_ERR_INVALID_ARGUMENT (metrics.cpp:38-39). */
hgs_status hgs_image_metrics(hgs_ctx *ctx, const void *gt, int dtype, int on_device, double *psnr_out,
                             double *ssim_out);
/* Standalone psnr / ssim (bindings.cpp:175-180) of two host images (h*w*3,
 * HGS_F64 or HGS_F32); NULL outputs are skipped. */
hgs_status hgs_metrics(hgs_ctx *ctx, const void *a, const void *b, int dtype, int width, int height,
                       double *psnr_out, double *ssim_out);
/* density_map: counts[h*w] = number of projected splats (dynamics only when
 * dynamics_only) whose clamped pixel box covers the pixel.  Releases the
 * last render's tape (it reuses the projection buffers). */
hgs_status hgs_density_map(hgs_ctx *ctx, const hgs_camera *cam, double t, int dynamics_only,
                           double weight_cutoff, uint32_t *counts_host);

/* ---- checkpoints (.hgsc, data_io.cpp:444-719) ---------- */
/* Versioned, CRC-32-checked, byte-identical to the reference's format.
 * Device scenes: the SCEN / OPTS payloads are encoded and decoded by CUDA
 * kernels straight from / into the FP32 SoA pools (FP32 widens exactly into
 * the f64 fields, so save -> load -> save is byte-identical); the host only
 * checksums and moves bytes.  Loading rounds f64 values to FP32 exactly like
 * hgs_scene_upload, validates quaternions (|q| within 1e-6 of 1) and flips
 * them to the canonical hemisphere (data_io.cpp:500-511).  A scene whose
 * Gaussians carry different SH degrees is a FormatError (the device pools
 * hold one degree).  Errors: HGS_ERR_FORMAT (bad magic, truncation,
 * trailing bytes, missing file, state/scene mismatch), HGS_ERR_INTEGRITY
 * (checksum), HGS_ERR_UNSUPPORTED_VERSION. */
hgs_status hgs_checkpoint_save(hgs_ctx *ctx, const char *path, int with_state);
/* Replaces the device scene (and, when the file has an OPTS section, the
 * optimizer state; otherwise it is zeroed).  has_state (optional) out. */
hgs_status hgs_checkpoint_load(hgs_ctx *ctx, const char *path, int *has_state);
/* Host scenes (bindings.cpp:197-205 save_checkpoint / load_checkpoint):
 * double precision, no device needed.  hgs_checkpoint_info validates the
 * whole file (checksums included) and returns the sizes to allocate;
 * hgs_checkpoint_read fills caller buffers (state_out may be NULL).  Errors
 * of these three are reported by hgs_io_last_error(). */
hgs_status hgs_checkpoint_write(const hgs_host_scene *scene, const hgs_host_state *state, const char *path);
hgs_status hgs_checkpoint_info(const char *path, int64_t *n4, int64_t *n3, int32_t *sh_degree, int *has_state);
hgs_status hgs_checkpoint_read(const char *path, hgs_host_scene *scene_out, hgs_host_state *state_out);
const char *hgs_io_last_error(void);

/* ---- initialisation (data_io.cpp:189-238) -------------- */
/* InitConfig (data_io.hpp:43-49) */
typedef struct {
    int32_t sh_degree;
    double tau, duration_seconds, init_temporal_scale, init_opacity;
} hgs_init_cfg;
/* init_scene: replaces the device scene with one dynamic Gaussian per point
 * (positions / rgb: n x 3 doubles), spatial log-scale from the mean distance
 * to the 3 nearest neighbours -- a tiled FP64 brute-force kNN on the GPU
 * instead of the reference's serial O(N^2) loop; extent = max distance to
 * the centroid.  n < 4 is HGS_ERR_INVALID_ARGUMENT (std::invalid_argument). */
hgs_status hgs_init_scene(hgs_ctx *ctx, const double *positions, const double *rgb, int64_t n,
                          const hgs_init_cfg *cfg);

/* ---- dataset frames: binary PPM (image.cpp:35-75) ------- */
/* Frames stay 8-bit sRGB (the HGS_U8 ground-truth dtype): hgs_ppm_read
 * copies the P6 payload (h*w*3 bytes) into `out` -- e.g. pinned memory
 * headed for the device -- with read_ppm's header rules and errors
 * (HGS_ERR_FORMAT: cannot open / not a P6 file / bad header / truncated
 * pixel data; a size other than width x height is a FormatError too).
 * hgs_ppm_read_batch reads n frames on `threads` host threads (0 = all
 * cores) and reports the first failing frame in order.  hgs_ppm_write
 * (write_ppm) quantises linear HGS_F64 / HGS_F32 images with
 * linear_to_srgb8 (image.cpp:15-18) or writes HGS_U8 codes as they are.
 * Context-free: errors are read with hgs_image_last_error(). */
hgs_status hgs_ppm_info(const char *path, int32_t *width, int32_t *height);
hgs_status hgs_ppm_read(const char *path, uint8_t *out, int32_t width, int32_t height);
hgs_status hgs_ppm_read_batch(const char *const *paths, int32_t n, uint8_t *const *outs, int32_t width,
                              int32_t height, int32_t threads);
hgs_status hgs_ppm_write(const char *path, const void *img, int dtype, int32_t width, int32_t height);
const char *hgs_image_last_error(void);

/* ---- optimizer (train.hpp:68-69) --------------------------------------- */
hgs_status hgs_adam_step(hgs_ctx *ctx, const hgs_lrs *lrs, double mean_lr_scale, int64_t *skipped_out);
hgs_status hgs_adam_state_download(hgs_ctx *ctx, hgs_host_scene *m, hgs_host_scene *v, int dtype,
                                   uint64_t *step);
hgs_status hgs_adam_state_upload(hgs_ctx *ctx, const hgs_host_scene *m, const hgs_host_scene *v, int dtype,
                                 uint64_t step);
hgs_status hgs_stats_download(hgs_ctx *ctx, double *grad_norm4, uint32_t *count4, double *grad_norm3,
                              uint32_t *count3);
/* Inverse of hgs_stats_download: GradAccum::grad_norm* / count*
 * (optim.hpp:32-41) into the device, pending deltas cleared. */
hgs_status hgs_stats_upload(hgs_ctx *ctx, const double *grad_norm4, const uint32_t *count4, const double *grad_norm3,
                            const uint32_t *count3);
/* Host gradients into the device gradient rows (layout of hgs_grads_download;
 * statistic deltas cleared), so a reference-signature optimizer_step(scene,
 * const SceneGrads&, ...) (train.hpp:68-69) runs hgs_adam_step on them. */
hgs_status hgs_grads_upload(hgs_ctx *ctx, const hgs_host_scene *grads, int dtype);
/* GradAccum::skipped_nonfinite (optim.hpp:39) of the device state: rows x
 * classes skipped for non-finite gradients since the upload; read (get)
 * and / or set it (set, e.g. when resuming from a checkpoint). */
hgs_status hgs_skipped_nonfinite(hgs_ctx *ctx, uint64_t *get, const uint64_t *set);

/* ---- conversion (scene.hpp:75 + train.cpp:305-362) --------------------- */
/* Moves every dynamic Gaussian with exp(s_t) > tau into the static pool
 * (stable), remaps the Adam rows and resets the densify statistics.
 * moved_out (optional, capacity n4) receives the converted indices. */
hgs_status hgs_sweep_convert(hgs_ctx *ctx, int64_t *moved_out, hgs_conversion_report *report);

/* ---- densification (train.cpp:182-299) ------------------ */
typedef struct {
    double grad_threshold, opacity_prune_eps, clone_size_frac, split_factor;
    int64_t max_gaussians; /* per pool */
} hgs_densify_cfg;
typedef struct {
    int64_t cloned3, split3, pruned3, cloned4, split4, pruned4; /* DensifyReport (train.hpp:73-77) */
    int64_t new_n3, new_n4;
} hgs_densify_report;
/* densify_and_prune in two calls, so the caller draws the reference's normal
 * variates (std::mt19937_64 + std::normal_distribution, in the reference's
 * order) between them:
 *   hgs_densify_plan: classifies on the device; kinds3/kinds4 (capacity n3 /
 *     n4) receive, in pool order, 1 = clone / 2 = split for every densified
 *     Gaussian; report has the counts and the new pool sizes.
 *   hgs_densify_apply: normals3 = 6 doubles per densified static (a clone
 *     uses the first 3 = one sample_normal3; a split two of them), normals4 =
 *     8 per densified dynamic (the Vec4 n as the reference builds it, twice
 *     for a split).  Rebuilds both pools (and the Adam moments: fresh rows
 *     zero), resets the densify statistics and gradients. */
hgs_status hgs_densify_plan(hgs_ctx *ctx, const hgs_densify_cfg *cfg, uint8_t *kinds3, uint8_t *kinds4,
                            hgs_densify_report *report);
hgs_status hgs_densify_apply(hgs_ctx *ctx, const double *normals3, const double *normals4, double split_factor);
/* The training loop's random stream (train.cpp:68-72, 245-275, 387-404):
 * libstdc++'s std::mt19937_64 with the reference's distributions, so batch
 * schedules and densification jitter match the reference bit for bit.
 *   hgs_rng_index       -- std::uniform_int_distribution<size_t>(lo, hi)
 *   hgs_rng_batch       -- `count` picks over [0, n_samples - 1] (one batch)
 *   hgs_densify_normals -- the normals for hgs_densify_apply given the kinds
 *                          hgs_densify_plan returned, drawn in the
 *                          reference's order
 *   hgs_densify_and_prune -- plan + draws + apply in one call (the
 *                          reference's densify_and_prune(scene, accum, cfg, rng)) */
typedef struct hgs_rng hgs_rng;
hgs_status hgs_rng_create(uint64_t seed, hgs_rng **out);
void hgs_rng_destroy(hgs_rng *rng);
uint64_t hgs_rng_raw(hgs_rng *rng);
uint64_t hgs_rng_index(hgs_rng *rng, uint64_t lo, uint64_t hi);
hgs_status hgs_rng_batch(hgs_rng *rng, uint64_t n_samples, int32_t count, uint64_t *out);
hgs_status hgs_densify_normals(hgs_rng *rng, const uint8_t *kinds3, int64_t d3, const uint8_t *kinds4, int64_t d4,
                               double *normals3, double *normals4);
hgs_status hgs_densify_and_prune(hgs_ctx *ctx, const hgs_densify_cfg *cfg, hgs_rng *rng,
                                 hgs_densify_report *report);
/* train.cpp:459-465: every opacity logit capped at floor_logit (logit(0.01)). */
hgs_status hgs_opacity_reset(hgs_ctx *ctx, double floor_logit);

/* ---- fused training iteration (train.cpp:402-475, one view batch) ------ */
typedef struct {
    double ssim_lambda;
    double weight_cutoff;
    double mean_lr_scale;
    hgs_lrs lrs;
    double bg[3];
} hgs_train_opts;
/* B views: render, loss against gt (device float images), backward scaled
 * by 1/batch_total, and (when apply_adam) one Adam step.  loss_out receives
 * the summed per-view loss.  A non-finite loss fails with
 * HGS_ERR_NUMERIC_ABORT when apply_adam (no update is applied); without the
 * update it is returned as is, for the caller to combine (e.g. the batch
 * loss summed over ranks) and decide. */
hgs_status hgs_train_step(hgs_ctx *ctx, int n_views, const hgs_camera *cams, const double *times,
                          const float *const *gt_device, int batch_total, const hgs_train_opts *opts,
                          int apply_adam, double *loss_out);

/* Same iteration with the ground-truth frames in HOST memory (dtype
 * HGS_F32/HGS_F64); the host->device copies run on the context stream
 * inside the call (the reference-facing end-to-end path). */
hgs_status hgs_train_step_host(hgs_ctx *ctx, int n_views, const hgs_camera *cams, const double *times,
                               const void *const *gt_host, int dtype, int batch_total, const hgs_train_opts *opts,
                               int apply_adam, double *loss_out);

/* Pipelined form of the same iteration (gt_on_device selects device float
 * frames or host frames of the given dtype): it is enqueued and the call
 * returns without waiting for it, so the host prepares iteration k+1 while
 * the device finishes iteration k.  hgs_train_collect returns the losses in
 * enqueue order.  A non-finite loss (train.cpp:445-447) makes the device skip
 * the Adam update of that iteration and of every later pending one; its
 * hgs_train_collect then fails with HGS_ERR_NUMERIC_ABORT and drops the
 * pending ones -- the parameters are those after the last finite iteration,
 * as when the reference throws.  At most HGS_TRAIN_PIPELINE iterations may be
 * pending (HGS_ERR_STATE otherwise); the synchronous entry points require an
 * empty pipeline. */
#define HGS_TRAIN_PIPELINE 4
hgs_status hgs_train_step_async(hgs_ctx *ctx, int n_views, const hgs_camera *cams, const double *times,
                                const void *const *gt, int dtype, int gt_on_device, int batch_total,
                                const hgs_train_opts *opts, int apply_adam);
hgs_status hgs_train_collect(hgs_ctx *ctx, double *loss_out);

/* Pipelined view-parallel iteration: after hgs_train_step_async(...,
 * apply_adam = 0) for this rank's views, hgs_train_exchange_async all-reduces
 * the loss-sum gate and the packed gradients and enqueues the Adam step gated
 * on the all-reduced loss (every rank skips a non-finite batch together) --
 * no host synchronisation; hgs_train_collect later returns this rank's loss
 * and raises NumericAbort on every rank for the same iteration. */
hgs_status hgs_train_exchange_async(hgs_ctx *ctx, const hgs_train_opts *opts);
/* Sharded optimizer exchange (enable = 1) for hgs_train_exchange_async:
 * instead of one all-reduce of the gradients and the full Adam step on every
 * rank, a reduce-scatter of every gradient row (rank r owns Gaussians
 * [r c, r c + c) of each pool, c = ceil(n / ranks) rounded up to 4), Adam on
 * the owned range only, and an all-gather of the updated parameter rows and
 * densification statistics -- the same bytes on the wire as the all-reduce,
 * 1/ranks of the Adam work.  The Adam moments then live sharded: before
 * anything that needs them whole (densification, the 4D->3D sweep,
 * checkpoints with state, hgs_adam_state_download, hgs_broadcast_params)
 * every rank calls hgs_gather_state (those calls fail with HGS_ERR_STATE
 * otherwise).  A one-rank communicator runs the same path (identity
 * collectives, the whole range). */
hgs_status hgs_comm_set_sharded(hgs_ctx *ctx, int enable);
hgs_status hgs_gather_state(hgs_ctx *ctx);
/* The shard [lo, hi) this rank owns of a pool of n Gaussians. */
void hgs_shard_range(int64_t n, int ranks, int rank, int64_t *lo, int64_t *hi);
/* Number of enqueued iterations not collected yet. */
int hgs_train_pending(hgs_ctx *ctx);

/* ---- instrumentation (not in the reference) ---------------------------- */
/* Per-phase CUDA-event timing on the context stream:
 * 0 preprocess, 1 depth sort, 2 duplicate, 3 tile sort, 4 raster fwd,
 * 5 loss, 6 raster bwd, 7 per-Gaussian bwd, 8 Adam, 9 sweep, 10 uploads. */
hgs_status hgs_profile(hgs_ctx *ctx, int enable);
hgs_status hgs_profile_read(hgs_ctx *ctx, double *ms16, long long *calls16, int reset);
/* Kernels launched by this library since load (process-wide). */
long long hgs_launch_count(void);
/* Parity introspection used by the tests: projected splats in projected
 * order (gid, f32 depth bits, box x0,x1,y0,y1, mean, conic, alpha, rgb) and
 * the tile-sorted instance list (tile id, gid) of the last render. */
hgs_status hgs_debug_splats(hgs_ctx *ctx, int32_t *gid, uint32_t *depth_bits, int32_t *box4, double *mean2,
                            double *conic4, double *alpha, float *rgb, int64_t cap, int64_t *n_out);
hgs_status hgs_debug_instances(hgs_ctx *ctx, uint32_t *tile, uint32_t *gid, int64_t cap, int64_t *n_out);
/* Parity introspection: the 8x8-quadrant contribution mask of every instance
 * of the kept full list, in hgs_debug_instances order. */
hgs_status hgs_debug_instance_masks(hgs_ctx *ctx, uint8_t *masks, int64_t cap, int64_t *n_out);
/* The rasterizers walk the exactly-culled instance list; keeping the
 * reference's complete list for hgs_debug_instances costs an extra sort. */
hgs_status hgs_debug_keep_instances(hgs_ctx *ctx, int enable);
/* Test hook: instance capacity of the next hgs_render_sweep frames. */
hgs_status hgs_debug_set_sweep_capacity(hgs_ctx *ctx, int64_t capacity);
/* Pixel-splat pair counters of the tile rasterizers (checked build
 * libhgs_gpu_checked.so only; HGS_ERR_STATE in the production library):
 * out[0..3] = K4 lane-iterations, box-covered pairs (exponent evaluated),
 * alpha-passing (composited) pairs, warp-iterations; out[4..7] the same for
 * K6.  reset != 0 zeroes them after the read. */
hgs_status hgs_debug_pair_counters(hgs_ctx *ctx, unsigned long long out[8], int reset);

#ifdef __cplusplus
}
#endif
#endif
