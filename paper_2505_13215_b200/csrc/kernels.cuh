// kernels.cuh -- declarations of the hot-path kernels (defined per .cu file).
#pragma once

#include "raster_common.cuh"

namespace hgs {

// preprocess.cu (K1)
__global__ void preprocess_kernel(const float* __restrict__ p4, int64_t cap4, int n4, const float* __restrict__ p3,
                                  int64_t cap3, int n3, int deg, DevCamera cam, double t, double cutoff, int tiles_x,
                                  SplatRec* __restrict__ rec, uint32_t* __restrict__ depth_key,
                                  uint32_t* __restrict__ ntiles_out, unsigned long long* __restrict__ stats,
                                  uint32_t* __restrict__ flags, ShRec* __restrict__ shrec);
// the same without the backward's ShRec (render-only frames)
__global__ void preprocess_render_kernel(const float* __restrict__ p4, int64_t cap4, int n4,
                                         const float* __restrict__ p3, int64_t cap3, int n3, int deg, DevCamera cam,
                                         double t, double cutoff, int tiles_x, SplatRec* __restrict__ rec,
                                         uint32_t* __restrict__ depth_key, uint32_t* __restrict__ ntiles_out,
                                         unsigned long long* __restrict__ stats, uint32_t* __restrict__ flags,
                                         ShRec* __restrict__ shrec);

size_t preprocess_smem_bytes(int deg);  // dynamic shared memory of a preprocess_kernel launch
cudaError_t preprocess_setup();         // opt-in to > 48 KB dynamic shared memory (once per process)

// raster_fwd.cu (K2 + K4)
__global__ void gather_sorted_kernel(const uint32_t* __restrict__ sorted_gid, const uint32_t* __restrict__ V_dev,
                                     const SplatRec* __restrict__ rec,
                                     const uint32_t* __restrict__ ntiles, SplatRec* __restrict__ rec_sorted,
                                     SplatFast* __restrict__ fast_sorted, uint32_t* __restrict__ ntiles_sorted,
                                     uint32_t* __restrict__ sorted_of_gid, CullRec* __restrict__ cull_rec);
constexpr int kDupPerCtaHost = 1024;  // instances per duplicate_kernel CTA
__global__ void duplicate_kernel(const SplatFast* __restrict__ fast, const SplatRec* __restrict__ exact, int V,
                                 const uint32_t* __restrict__ offsets, int tiles_x, int cull,
                                 const CullRec* __restrict__ cull_rec, uint32_t* __restrict__ keys,
                                 uint32_t* __restrict__ vals, uint32_t* __restrict__ keep,
                                 const uint32_t* __restrict__ cta_first, int I);
__global__ void duplicate_compact_kernel(const SplatFast* __restrict__ fast, int V, const uint32_t* __restrict__ offsets,
                                         int tiles_x, const CullRec* __restrict__ cull_rec,
                                         const uint32_t* __restrict__ cta_first, int I, uint32_t* __restrict__ keys_out,
                                         uint32_t* __restrict__ vals_out, uint32_t* __restrict__ kept_total,
                                         unsigned long long* status, uint32_t* __restrict__ counter,
                                         const uint32_t* V_dev, const uint32_t* I_dev, uint32_t* flags);
__global__ void dup_bounds_kernel(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ ntiles_sorted,
                                  int V, uint32_t* __restrict__ cta_first, const uint32_t* V_dev, uint32_t nblocks,
                                  uint32_t* __restrict__ zero_words, uint32_t n_zero);
__global__ void compact_instances_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, int n,
                                         const uint32_t* __restrict__ pos, uint32_t* __restrict__ keys_out,
                                         uint32_t* __restrict__ vals_out);
__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, int n, uint2* __restrict__ ranges);
__global__ void tile_ranges_dev_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ n_dev,
                                       uint2* __restrict__ ranges);
void set_debug_exact(int v);  // raster_fwd.cu (HGS_DEBUG_EXACT diagnostics)
void set_debug_terr(float v);
void launch_raster_fwd(bool count_map, int n_tiles, cudaStream_t st, const uint2* ranges, const uint32_t* inst_val,
                       const SplatFast* fast, const SplatRec* exact, int W, int H, int tiles_x, float bg_r, float bg_g,
                       float bg_b, float* out_rgb, uint32_t* out_last, float* out_tfinal, float* out_trans,
                       uint32_t* out_count, uint32_t* fix_list, uint32_t* fix_count, uint32_t* tile_order,
                       double bg_rd, double bg_gd, double bg_bd, double* out_cout, uint32_t* fix_slot,
                       const uint32_t* remap = nullptr);


__global__ void grads_pack_kernel(const float* __restrict__ gbuf, int64_t off_g3, int64_t off_dgn4, int rows4,
                                  int rows3, int64_t cap4, int64_t cap3, int n4, int n3, float* __restrict__ packed,
                                  int unpack);
// K7b: SH colour backward (runs before K7)
__global__ void sh_bwd_kernel(int N, const uint32_t* __restrict__ sorted_of_gid, const acc_t* __restrict__ accum,
                              int acc_stride, int n4, const float* __restrict__ p4, int64_t cap4,
                              const float* __restrict__ p3, int64_t cap3, int deg, float scale,
                              float* __restrict__ g4, float* __restrict__ g3, const ShRec* __restrict__ shrec,
                              float4* __restrict__ ddir, int first);

}  // namespace hgs

namespace hgs {

// raster_bwd.cu (K6)

__global__ void raster_bwd_kernel(const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val,
                                  const SplatFast* __restrict__ fast, const SplatRec* __restrict__ exact, int W, int H,
                                  int tiles_x, const float* __restrict__ tfinal, const uint32_t* __restrict__ last_arr,
                                  const float* __restrict__ dL_dimg, float bg_r, float bg_g, float bg_b,
                                  acc_t* __restrict__ accum, const uint32_t* __restrict__ tile_order,
                                  const uint32_t* __restrict__ fix_slot, const double* __restrict__ fix_cout,
                                  double bg_rd, double bg_gd, double bg_bd);
__global__ void raster_bwd_exact_kernel(int all_pixels, const uint2* __restrict__ ranges,
                                        const uint32_t* __restrict__ inst_val, const SplatRec* __restrict__ exact,
                                        int W, int tiles_x, double bg_r, double bg_g, double bg_b,
                                        const uint32_t* __restrict__ last_arr, const float* __restrict__ dL_dimg,
                                        const double* __restrict__ col64, acc_t* __restrict__ accum);
__global__ void exact_colour_kernel(const uint32_t* __restrict__ sorted_gid, int V, int n4,
                                    const float* __restrict__ p4, int64_t cap4, const float* __restrict__ p3,
                                    int64_t cap3, int deg, DevCamera cam, double t, double* __restrict__ col64);
// gaussian_bwd.cu (K7)
__global__ void gaussian_bwd_kernel(int N, const uint32_t* __restrict__ sorted_of_gid, const acc_t* __restrict__ accum,
                                    int acc_stride, int n4, const float* __restrict__ p4, int64_t cap4,
                                    const float* __restrict__ p3, int64_t cap3, int deg, DevCamera cam, double t,
                                    double scale, float* __restrict__ g4, float* __restrict__ g3,
                                    float* __restrict__ sn4, float* __restrict__ sn3, float* __restrict__ gn4,
                                    float* __restrict__ gn3, float* __restrict__ cnt4, float* __restrict__ cnt3,
                                    const double* __restrict__ conic_src, int conic_stride, const float4* __restrict__ ddir, int first);
__global__ void gaussian_bwd_exact_kernel(int N, const uint32_t* __restrict__ sorted_of_gid, const acc_t* __restrict__ accum,
                                    int acc_stride, int n4, const float* __restrict__ p4, int64_t cap4,
                                    const float* __restrict__ p3, int64_t cap3, int deg, DevCamera cam, double t,
                                    double scale, float* __restrict__ g4, float* __restrict__ g3,
                                    float* __restrict__ sn4, float* __restrict__ sn3, float* __restrict__ gn4,
                                    float* __restrict__ gn3, float* __restrict__ cnt4, float* __restrict__ cnt3,
                                    const double* __restrict__ conic_src, int conic_stride, const float4* __restrict__ ddir, int first);
// loss.cu (K5)
void set_ssim_window();
void set_srgb_lut();
void launch_loss(cudaStream_t st, const float* img, const void* gt, bool gt_u8, int W, int H, float* maps,
                 float lambda, bool with_ssim, float* grad, double* sums);
void launch_metrics(cudaStream_t st, const float* img, const void* gt, bool gt_u8, int W, int H, float* maps,
                    double* sums);
// density_map (raster.cpp:268-287): +1 over every projected splat's box via a
// 2D difference array and row / column prefix sums
__global__ void density_diff_kernel(const uint32_t* __restrict__ ntiles, const SplatRec* __restrict__ rec, int n,
                                    int W, int H, int* __restrict__ diff);
__global__ void density_rows_kernel(int* __restrict__ diff, int W, int H);
__global__ void density_cols_kernel(const int* __restrict__ diff, int W, int H, uint32_t* __restrict__ out);
// adam.cu (K8)
struct AdamArgs {
    float b1, b2, one_m_b1, one_m_b2;
    float inv_bc1, inv_bc2;
    float lr_mean, lr_mean_t, lr_quat, lr_scales, lr_opacity, lr_sh;
    const double* view_sums = nullptr;  // the step's (ssim, l1) loss sums per view
    int n_views = 0;                    // > 0: skip the whole update if one is non-finite
    uint32_t* abort = nullptr;          // sticky: set by a non-finite step, blocks later updates
    unsigned long long* skipped_cum = nullptr;  // GradAccum::skipped_nonfinite (never reset by a step)
};
struct AdamPools {
    float *p4, *g4, *m4, *v4, *p3, *g3, *m3, *v3;
    float *gn4, *cnt4, *dgn4, *dcnt4, *gn3, *cnt3, *dgn3, *dcnt3;
    int64_t cap4, cap3;
    int n4, n3, K3;  // K3 = 3 * sh_count(deg)
};
// Threads per 4 Gaussians checking the SH class's gradient rows (K3 rows)
__host__ __device__ inline int adam_sh_slices(int K3) { return K3 >= 16 ? 4 : 1; }
// adam_classes_kernel's thread count
inline uint32_t adam_class_units(int n3, int n4, int K3) {
    const uint32_t q3 = div_up((uint32_t)n3, 4), q4 = div_up((uint32_t)n4, 4), S = adam_sh_slices(K3);
    return (4 + S) * q3 + ((6 * q4 + 3) & ~3u) + S * q4;
}
__global__ void adam_classes_kernel(AdamPools P, AdamArgs A, uint8_t* __restrict__ cls_ok3,
                                    uint8_t* __restrict__ cls_ok4, unsigned long long* __restrict__ skipped_total,
                                    uint32_t* __restrict__ flags);
__global__ void adam_rows_kernel(AdamPools P, AdamArgs A, const uint8_t* __restrict__ cls_ok3,
                                 const uint8_t* __restrict__ cls_ok4, int blocks_per_row3, int blocks_per_row4);
// convert.cu (K9)
__global__ void convert_mask_kernel(const float* __restrict__ p4, int64_t cap4, int n4, double s_star,
                                    uint32_t* __restrict__ mask);
__global__ void convert_rows_kernel(const float* __restrict__ p4, const float* __restrict__ m4,
                                    const float* __restrict__ v4, int64_t cap4, int n4,
                                    const uint32_t* __restrict__ mask, const uint32_t* __restrict__ pos,
                                    float* __restrict__ p3, float* __restrict__ m3, float* __restrict__ v3,
                                    int64_t cap3, int n3, int deg, long long* __restrict__ moved,
                                    unsigned long long* __restrict__ max_leak_bits, double* __restrict__ leak_sum,
                                    uint32_t* __restrict__ flags);
__global__ void compact_survivors_kernel(const float* __restrict__ src, float* __restrict__ dst, int rows,
                                         int64_t cap4, int n4, const uint32_t* __restrict__ mask,
                                         const uint32_t* __restrict__ pos);

__global__ void grads_pack_kernel(const float* __restrict__ gbuf, int64_t off_g3, int64_t off_dgn4, int rows4,
                                  int rows3, int64_t cap4, int64_t cap3, int n4, int n3, float* __restrict__ packed,
                                  int unpack);
// K7b: SH colour backward (runs before K7)
__global__ void sh_bwd_kernel(int N, const uint32_t* __restrict__ sorted_of_gid, const acc_t* __restrict__ accum,
                              int acc_stride, int n4, const float* __restrict__ p4, int64_t cap4,
                              const float* __restrict__ p3, int64_t cap3, int deg, float scale,
                              float* __restrict__ g4, float* __restrict__ g3, const ShRec* __restrict__ shrec,
                              float4* __restrict__ ddir, int first);

}  // namespace hgs
