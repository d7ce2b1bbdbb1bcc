// kernels.cuh -- declarations of the hot-path kernels (defined per .cu file).
#pragma once

#include "raster_common.cuh"

namespace hgs {

// preprocess.cu (K1)
__global__ void preprocess_kernel(const float* __restrict__ p4, int64_t cap4, int n4, const float* __restrict__ p3,
                                  int64_t cap3, int n3, int deg, DevCamera cam, double t, double cutoff, int tiles_x,
                                  SplatRec* __restrict__ rec, uint32_t* __restrict__ depth_key,
                                  uint32_t* __restrict__ ntiles_out, unsigned long long* __restrict__ stats,
                                  uint32_t* __restrict__ flags);

// raster_fwd.cu (K2 + K4)
__global__ void gather_sorted_kernel(const uint32_t* __restrict__ sorted_gid, int V, const SplatRec* __restrict__ rec,
                                     const uint32_t* __restrict__ ntiles, SplatRec* __restrict__ rec_sorted,
                                     SplatFast* __restrict__ fast_sorted, uint32_t* __restrict__ ntiles_sorted);
__global__ void duplicate_kernel(const SplatFast* __restrict__ fast, int V, const uint32_t* __restrict__ offsets,
                                 int tiles_x, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals);
__global__ void tile_ranges_kernel(const uint32_t* __restrict__ keys, int n, uint2* __restrict__ ranges);
__global__ void raster_fwd_kernel(const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val,
                                  const SplatFast* __restrict__ fast, const SplatRec* __restrict__ exact, int W, int H,
                                  int tiles_x, float bg_r, float bg_g, float bg_b, float* __restrict__ out_rgb,
                                  uint32_t* __restrict__ out_last, float* __restrict__ out_trans,
                                  uint32_t* __restrict__ out_count, uint32_t* __restrict__ fix_list,
                                  uint32_t* __restrict__ fix_count);
__global__ void raster_fixup_kernel(const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ fix_count,
                                    const uint2* __restrict__ ranges, const uint32_t* __restrict__ inst_val,
                                    const SplatRec* __restrict__ exact, int W, int tiles_x, double bg_r, double bg_g,
                                    double bg_b, float* __restrict__ out_rgb, uint32_t* __restrict__ out_last,
                                    float* __restrict__ out_trans, uint32_t* __restrict__ out_count);

}  // namespace hgs
