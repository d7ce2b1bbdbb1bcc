// primitives.cuh -- device-wide scan / radix sort (see primitives.cu)
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hgs_common.cuh"

namespace hgs {

size_t scan_workspace_bytes(int n);
// out[i] = sum(in[0..i)); *total (device, optional) = sum(in)
// n_dev (optional): device-side item count (then n is ignored).  in may equal out.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int n, uint32_t* total, uint32_t* ws,
                        cudaStream_t st, const uint32_t* n_dev = nullptr);

// keys[r] = depth_key[i], vals[r] = i for the i with ntiles[i] > 0, in index
// order; *total (device) = their count.  ws: scan_workspace_bytes(n).
void compact_visible(const uint32_t* ntiles, const uint32_t* depth_key, int n, uint32_t* keys, uint32_t* vals,
                     uint32_t* total, uint32_t* ws, cudaStream_t st);

size_t radix_workspace_bytes(int n);
// n_dev (optional): device-side item count (then n is ignored).  ranges
// (optional): [first, end) of every key's run in the sorted keys (the tile
// ranges; entries of absent keys untouched).
int radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int n,
                     int begin_bit, int end_bit, uint32_t* ws, cudaStream_t st, const uint32_t* n_dev = nullptr,
                     uint2* ranges = nullptr);

}  // namespace hgs
