/*
 * hgs_oracle.h -- C ABI of the CPU FP64 oracle (TEST INFRASTRUCTURE ONLY).
 *
 * This library restates, in plain double-precision C++, the reference's
 * render-and-train hot path (/root/reference/proj).
 * It exists so that tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs can check and time the CUDA product.
 * Nothing in paper_2505_13215_b200/ may link or call it.
 *
 * Parity status: PINNED against the reference itself.  oracle/_ref is the
 * reference's own proj/src compiled here from its sources against
 * self-written Eigen / doctest stand-ins (oracle/ref_shim; Eigen3 and
 * doctest are not installed), with a C ABI in these struct types
 * (oracle/ref_capi.cpp).  The reference's 70 doctest cases pass against that
 * build, and on the oracle's fixtures the two agree bit for bit on images,
 * transmittance / count maps, RenderStats, every projected splat, the Adam
 * updates and the checkpoint bytes, and to summation-order rounding (1e-12)
 * on gradients and the conversion sweep (tests/test_oracle_vs_reference.py;
 * reference-produced fixtures in tests/golden/ref_golden.npz keep the pin
 * where /root/reference is absent).  Remaining boundary: the stand-in's
 * arithmetic order is left-to-right, Eigen's own is not observable here
 * (third-party arithmetic), and its eigen-solver / SVD are
 * Jacobi iterations meeting Eigen's contracts, not Eigen's algorithms.
 */
#ifndef HGS_ORACLE_H
#define HGS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene pools, row-major per parameter class (reference scene.hpp:13-59).
 * K = (sh_degree+1)^2 SH coefficients, each an RGB triple (sh.hpp:15-22). */
typedef struct {
    int64_t n4, n3;
    int32_t sh_degree;
    double tau, extent;
    /* dynamics (Gaussian4D) */
    double *mean_x;  /* [n4*3] */
    double *mean_t;  /* [n4]   */
    double *ql;      /* [n4*4] (w,x,y,z) */
    double *qr;      /* [n4*4] */
    double *log_s4;  /* [n4*4] (s_x,s_y,s_z,s_t) */
    double *op4;     /* [n4]   opacity logit */
    double *sh4;     /* [n4*K*3] */
    /* statics (Gaussian3D) */
    double *mean3;   /* [n3*3] */
    double *quat3;   /* [n3*4] */
    double *log_s3;  /* [n3*3] */
    double *op3;     /* [n3]   */
    double *sh3;     /* [n3*K*3] */
} hgso_scene;

/* Gradients, same layout as the scene plus screen_norm (backward.hpp:13-31). */
typedef struct {
    double *mean_x, *mean_t, *ql, *qr, *log_s4, *op4, *sh4, *screen_norm4;
    double *mean3, *quat3, *log_s3, *op3, *sh3, *screen_norm3;
} hgso_grads;

/* Pinhole camera (camera.hpp:11-16); rot row-major, x_cam = R x + t. */
typedef struct {
    double fx, fy, cx, cy;
    double rot[9];
    double trans[3];
    int32_t width, height;
    double near_, far_;
} hgso_camera;

/* RenderStats (raster.hpp:33-40) */
typedef struct {
    int64_t culled_depth, culled_offscreen, culled_degenerate, culled_temporal,
        degenerate_temporal, projected;
} hgso_stats;

/* One projected splat (SplatPrimitive, raster.hpp:22-31) + its clamped box. */
typedef struct {
    double sx, sy;
    double conic[4];
    double depth;
    double rgb[3];
    double alpha;
    int32_t radius;
    int32_t pool;   /* 0 statics, 1 dynamics */
    int32_t index;  /* pool index */
    int32_t gid;    /* dynamics: index; statics: n4 + index */
    int32_t x0, x1, y0, y1;
    uint32_t depth_bits;
    int32_t pad_;
} hgso_splat;

/* Adam state: m and v laid out exactly like the scene params. */
typedef struct {
    hgso_scene m, v;           /* only the pointer fields are used */
    double *grad_norm4, *grad_norm3;
    uint32_t *count4, *count3;
    uint64_t step;
    uint64_t skipped_nonfinite;
} hgso_state;

typedef struct {
    double mean, mean_final_ratio, mean_t, quat, scales, opacity, sh;
} hgso_lrs;

typedef struct {
    int64_t count;
    double max_leakage, mean_leakage;
} hgso_conversion;

/* densify_and_prune configuration (train.hpp:23-49 fields it reads) and report */
typedef struct {
    double grad_threshold, opacity_prune_eps, clone_size_frac, split_factor;
    int64_t max_gaussians;
} hgso_densify_cfg;

typedef struct {
    int64_t cloned3, split3, pruned3, cloned4, split4, pruned4;
} hgso_densify_report;

/* status codes: 0 ok; the message is in hgso_last_error() */
enum {
    HGSO_OK = 0,
    HGSO_INVALID_ARGUMENT = 1,
    HGSO_DEGENERATE_TEMPORAL = 2,
    HGSO_DEGENERATE_ROTATION = 3,
    HGSO_NUMERIC_ABORT = 4,
};

const char *hgso_last_error(void);

/* --- fixtures (tests/oracles.hpp:26-108), libstdc++ mt19937_64 ------------- */
void *hgso_rng_new(uint64_t seed);
void hgso_rng_free(void *rng);
double hgso_rng_uniform(void *rng);  /* uniform_real_distribution(0,1) */
double hgso_rng_normal(void *rng);   /* a fresh normal_distribution(0,1) draw */
uint64_t hgso_rng_index(void *rng, uint64_t lo, uint64_t hi); /* uniform_int_distribution<size_t>(lo, hi) */
uint64_t hgso_rng_raw(void *rng);    /* one raw mt19937_64 output */
/* n draws from ONE std::normal_distribution(0,1) object (its cached second
 * polar value carries across the draws) */
void hgso_rng_normal_seq(void *rng, int64_t n, double *out);
/* densify_and_prune (train.cpp:182-299): in -> out (out arrays sized by the
 * caller for the worst case, out->n3/n4 set), Adam m/v remapped (fresh rows
 * zero), statistics reset; the rng is advanced exactly like the reference. */
int hgso_densify_and_prune(const hgso_scene *in, const hgso_state *st_in, hgso_scene *out, hgso_state *st_out,
                           const hgso_densify_cfg *cfg, void *rng, hgso_densify_report *rep);
/* init_scene (data_io.cpp:189-238): out sized for n dynamics, no statics */
int hgso_init_scene(const double *pos, const double *rgb, int64_t n, int sh_degree, double tau, double duration,
                    double init_temporal_scale, double init_opacity, hgso_scene *out, double *duration_out);
/* random_scene: caller passes buffers sized for (n_static, n_dynamic, degree) */
void hgso_random_scene(void *rng, int n_static, int n_dynamic, int sh_degree, hgso_scene *out);
void hgso_random_quat(void *rng, double q[4]);
int hgso_random_camera(void *rng, int width, int height, hgso_camera *out);
int hgso_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                 int width, int height, hgso_camera *out);

/* --- math kernels (gauss_math.cpp) -------------------------------------- */
int hgso_quat_to_rot3(const double q[4], double r[9]);
int hgso_rot3_to_quat(const double r[9], double q[4]);
void hgso_rot4_from_pair(const double ql[4], const double qr[4], double r[16]);
void hgso_build_cov4(const double r[16], const double log_s[4], double cov[16]);
void hgso_build_cov3(const double r[9], const double log_s[3], double cov[9]);
int hgso_condition_at_time(const double mean4[4], const double cov4[16], double t,
                           double mean3[3], double cov3[9], double *weight);
int hgso_clamp_psd(const double m[9], double eps, double out[9]);
int hgso_extract_spatial_rot(const double r4[16], double r3[9], double *leakage);
void hgso_sh_basis(const double dir[3], int degree, double out[16]);
void hgso_sh_basis_grad(const double dir[3], int degree, double out[48]);
int hgso_eval_sh(const double *coeffs, int degree, const double dir[3], double rgb[3]);
double hgso_exp(double x);

/* --- renderer (raster.cpp) ----------------------------------------------- */
/* project_3d (raster.cpp:26-64): returns 1 and fills *out when projected */
int hgso_project_3d(const double mean3[3], const double cov3[9], const hgso_camera *cam,
                    hgso_splat *out, hgso_stats *stats, int *projected);
/* density_map (raster.cpp:268-287): counts[h*w] */
int hgso_density_map(const hgso_scene *s, const hgso_camera *cam, double t, int dynamics_only, double weight_cutoff,
                     uint32_t *counts);
/* project_scene: writes up to cap splats (dynamics first, then statics) */
int hgso_project_scene(const hgso_scene *s, const hgso_camera *cam, double t, double weight_cutoff,
                       hgso_splat *out, int64_t cap, int64_t *n_out, hgso_stats *stats);
/* sorted instance list: tile ids and projected-prim indices in (key, prim) order */
int hgso_sorted_instances(const hgso_scene *s, const hgso_camera *cam, double t,
                          double weight_cutoff, uint32_t *tile_out, uint32_t *prim_out,
                          int64_t cap, int64_t *n_out);
int hgso_rasterize(const hgso_scene *s, const hgso_camera *cam, double t, const double bg[3],
                   double weight_cutoff, int num_threads, double *rgb_out, uint32_t *count_out,
                   double *trans_out, hgso_stats *stats);
int hgso_reference_render(const hgso_scene *s, const hgso_camera *cam, double t,
                          const double bg[3], double weight_cutoff, double *rgb_out,
                          hgso_stats *stats);

/* --- differentiable forward / backward (backward.cpp) -------------------- */
/* tiled forward with tape (bitwise == rasterize); returns an opaque tape */
int hgso_forward_train(const hgso_scene *s, const hgso_camera *cam, double t, const double bg[3],
                       double weight_cutoff, int num_threads, double *rgb_out, void **tape_out);
/* the literal untiled forward_train (backward.cpp:89-176), small sizes only */
int hgso_forward_train_untiled(const hgso_scene *s, const hgso_camera *cam, double t,
                               const double bg[3], double weight_cutoff, double *rgb_out,
                               void **tape_out);
void hgso_tape_free(void *tape);
int64_t hgso_tape_contrib_total(void *tape);
/* accumulates into g (which must be zero-initialised / sized like the scene) */
int hgso_backward(const hgso_scene *s, const hgso_camera *cam, void *tape, const double *loss_grad,
                  hgso_grads *g);
void hgso_grads_add_scaled(const hgso_scene *shape, hgso_grads *acc, const hgso_grads *other,
                           double scale);

/* --- loss / metrics (loss.cpp, metrics.cpp) ------------------------------ */
double hgso_photometric_loss(const double *a, const double *b, int w, int h, double lambda);
double hgso_photometric_loss_with_grad(const double *a, const double *b, int w, int h,
                                       double lambda, double *grad);
double hgso_ssim(const double *a, const double *b, int w, int h);
double hgso_ssim_with_grad(const double *a, const double *b, int w, int h, double *grad);
double hgso_psnr(const double *a, const double *b, int w, int h);

/* --- optimizer (train.cpp:18-180) ---------------------------------------- */
int hgso_optimizer_step(hgso_scene *s, const hgso_grads *g, hgso_state *st, const hgso_lrs *lrs,
                        double mean_lr_scale);
/* densify statistics from one image's grads (train.cpp:433-444) */
void hgso_accumulate_stats(const hgso_scene *shape, hgso_state *st, const hgso_grads *g);

/* --- conversion (scene.cpp:10-71 + train.cpp:305-362) -------------------- */
int hgso_is_static(double log_st, double tau, int *out);
/* In-place sweep: pools and state are compacted; dst buffers must have room
 * for n3 + n4 statics.  moved receives the converted dynamics indices. */
int hgso_sweep_convert(hgso_scene *s, hgso_state *st, int64_t *moved, hgso_conversion *rep);
int hgso_convert_4d_to_3d(const double mean_x[3], double mean_t, const double ql[4],
                          const double qr[4], const double log_s4[4], double op,
                          double mean3[3], double quat3[4], double log_s3[3], double *op3);

/* --- one training iteration (train.cpp:402-450) -------------------------- */
int hgso_train_step(hgso_scene *s, hgso_state *st, const hgso_camera *cams, const double *times,
                    const double *const *gts, int n_views, const double bg[3], double weight_cutoff,
                    double ssim_lambda, const hgso_lrs *lrs, double mean_lr_scale, int num_threads,
                    int tile_threads, double *loss_out);

int hgso_hardware_threads(void);

#ifdef __cplusplus
}
#endif
#endif
