// primitives.cu -- device-wide exclusive scan and stable LSD radix sort.
//
// Hand-written for sm_100a (no CUB on the product path).  The radix sort is
// the stable key/value sort the reference's std::sort over (key, prim)
// (raster.cpp:202) reduces to: instances are emitted in projected-index order,
// sorted once by f32 depth bits (4 x 8-bit passes) and then by tile id
// (ceil(bits/8) passes); stability carries the index tie-break through both.
//
// Each pass = per-block digit histogram (shared-memory atomics), one
// exclusive scan of the digit-major histogram, and a scatter that ranks
// items stably inside each warp with __match_any_sync + per-warp counters.
#include <cstdio>

#include "primitives.cuh"

namespace hgs {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

__device__ inline uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread.
template <int NT>
__device__ inline void block_excl_scan(uint32_t v, uint32_t& excl) {
    __shared__ uint32_t warp_tot[NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = warp_incl_scan(v);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? warp_tot[lane] : 0u;
        uint32_t wi = warp_incl_scan(w);
        if (lane < NT / 32) warp_tot[lane] = wi - w;
    }
    __syncthreads();
    excl = incl - v + warp_tot[warp];
    __syncthreads();
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const uint32_t* __restrict__ in, int n,
                                                                   uint32_t* __restrict__ block_sums) {
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += (base + k < n) ? in[base + k] : 0u;
    __shared__ uint32_t red[kScanThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += red[w];
        block_sums[blockIdx.x] = t;
    }
}

// Single-block exclusive scan of up to 1024*kScanItems values, in place.
__global__ void __launch_bounds__(1024) scan_single_kernel(uint32_t* __restrict__ data, int n,
                                                           uint32_t* __restrict__ total) {
    const int base = threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? data[base + k] : 0u;
        s += v[k];
    }
    uint32_t excl;
    block_excl_scan<1024>(s, excl);
    uint32_t run = excl;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) data[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == 1023 && total) *total = excl + s;
}

__global__ void __launch_bounds__(kScanThreads) scan_downsweep_kernel(const uint32_t* __restrict__ in, int n,
                                                                      const uint32_t* __restrict__ block_off,
                                                                      uint32_t* __restrict__ out) {
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < n) ? in[base + k] : 0u;
        s += v[k];
    }
    uint32_t excl;
    block_excl_scan<kScanThreads>(s, excl);
    uint32_t run = excl + block_off[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

// ---------------------------------------------------------------- radix sort
constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096
constexpr int kSortWarps = kSortThreads / 32;

__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const uint32_t* __restrict__ keys, int n,
                                                                  int shift, int nblocks,
                                                                  uint32_t* __restrict__ hist,
                                                                  const uint32_t* __restrict__ n_dev) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    if (n_dev) n = (int)*n_dev;
    const int base = blockIdx.x * kSortTile;
#pragma unroll 4
    for (int k = 0; k < kSortItems; ++k) {
        const int idx = base + k * kSortThreads + threadIdx.x;
        if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, int n, int shift, int nblocks, const uint32_t* __restrict__ offsets,
    const uint32_t* __restrict__ n_dev) {
    __shared__ uint32_t cnt[kSortWarps][256];
    __shared__ uint32_t goff[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (n_dev) n = (int)*n_dev;
    if ((int)(blockIdx.x * kSortTile) >= n) return;  // whole block beyond the device-side count
    for (int i = threadIdx.x; i < kSortWarps * 256; i += kSortThreads) (&cnt[0][0])[i] = 0u;
    goff[threadIdx.x] = offsets[threadIdx.x * nblocks + blockIdx.x];
    __syncthreads();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int base = blockIdx.x * kSortTile + warp * (kSortItems * 32);
    uint32_t k[kSortItems], v[kSortItems], rank[kSortItems];
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int idx = base + r * 32 + lane;
        const bool valid = idx < n;
        k[r] = valid ? keys[idx] : 0u;
        v[r] = valid ? vals[idx] : 0u;
        const uint32_t d = valid ? ((k[r] >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t before = valid ? cnt[warp][d] : 0u;
        __syncwarp();
        if (valid && lane == __ffs(peers) - 1) cnt[warp][d] = before + __popc(peers);
        __syncwarp();
        rank[r] = before + __popc(peers & lt_mask);
    }
    __syncthreads();
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortWarps; ++w) {
            const uint32_t t = cnt[w][threadIdx.x];
            cnt[w][threadIdx.x] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kSortItems; ++r) {
        const int idx = base + r * 32 + lane;
        if (idx < n) {
            const uint32_t d = (k[r] >> shift) & 255u;
            const uint32_t pos = goff[d] + cnt[warp][d] + rank[r];
            keys_out[pos] = k[r];
            vals_out[pos] = v[r];
        }
    }
}

}  // namespace

size_t scan_workspace_bytes(int n) {
    const int nb = (int)div_up((uint32_t)n, kScanTile);
    return (size_t)(nb + 32) * sizeof(uint32_t);
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int n, uint32_t* total, uint32_t* ws,
                        cudaStream_t st) {
    if (n <= 0) {
        if (total) cudaMemsetAsync(total, 0, sizeof(uint32_t), st);
        return;
    }
    if (n <= 1024 * kScanItems) {  // one CTA: a single launch
        if (in != out) cudaMemcpyAsync(out, in, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
        scan_single_kernel<<<1, 1024, 0, st>>>(out, n, total);
        count_launch();
        return;
    }
    const int nb = (int)div_up((uint32_t)n, kScanTile);
    if (nb > 1024 * kScanItems) {
        fprintf(stderr, "exclusive_scan_u32: n=%d exceeds the single-level capacity\n", n);
        return;
    }
    scan_reduce_kernel<<<nb, kScanThreads, 0, st>>>(in, n, ws);
    count_launch();
    scan_single_kernel<<<1, 1024, 0, st>>>(ws, nb, total);
    count_launch();
    scan_downsweep_kernel<<<nb, kScanThreads, 0, st>>>(in, n, ws, out);
    count_launch();
}

size_t radix_workspace_bytes(int n) {
    const int nb = (int)div_up((uint32_t)n, kSortTile);
    const size_t hist = (size_t)256 * nb;
    return (hist * 2 + 64) * sizeof(uint32_t) + scan_workspace_bytes((int)hist);
}

// Stable LSD sort of (keys, vals) on bits [begin_bit, end_bit).  The result
// lands in (keys, vals) when the pass count is even, else in (keys_alt,
// vals_alt); the return value says which (0 = original buffers).
int radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int n,
                     int begin_bit, int end_bit, uint32_t* ws, cudaStream_t st, const uint32_t* n_dev) {
    if (n <= 1 && !n_dev) return 0;
    if (n < 1) return 0;
    const int nb = (int)div_up((uint32_t)n, kSortTile);
    const int hist_n = 256 * nb;
    uint32_t* hist = ws;
    uint32_t* offs = ws + hist_n;
    uint32_t* scan_ws = offs + hist_n + 64;
    int cur = 0;
    uint32_t* kin = keys;
    uint32_t* vin = vals;
    uint32_t* kout = keys_alt;
    uint32_t* vout = vals_alt;
    for (int shift = begin_bit; shift < end_bit; shift += 8) {
        radix_hist_kernel<<<nb, kSortThreads, 0, st>>>(kin, n, shift, nb, hist, n_dev);
        count_launch();
        exclusive_scan_u32(hist, offs, hist_n, nullptr, scan_ws, st);
        radix_scatter_kernel<<<nb, kSortThreads, 0, st>>>(kin, vin, kout, vout, n, shift, nb, offs, n_dev);
        count_launch();
        uint32_t* t = kin;
        kin = kout;
        kout = t;
        t = vin;
        vin = vout;
        vout = t;
        cur ^= 1;
    }
    return cur;
}

}  // namespace hgs

#include <atomic>
namespace hgs {
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
}  // namespace hgs
