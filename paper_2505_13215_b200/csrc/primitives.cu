// primitives.cu -- device-wide exclusive scan and stable LSD radix sort.
//
// Hand-written for sm_100a (no CUB on the product path).  The radix sort is
// the stable key/value sort the reference's std::sort over (key, prim)
// (raster.cpp:202) reduces to: instances are emitted in projected-index order,
// sorted once by f32 depth bits (4 x 8-bit passes) and then by tile id
// (ceil(bits/8) passes); stability carries the index tie-break through both.
//
// Both are ONE cooperative launch (persistent grid, co-resident by
// construction, grid-wide barriers between phases) so a whole sort or scan
// costs one launch instead of 3-5 per pass: every block owns one contiguous,
// ordered chunk of the items.
//   scan:  block sums | barrier | prefix of the preceding block sums + block
//          scans of the chunk in 4096-item tiles.
//   sort pass: chunk digit histogram -> [digit][block] | barrier | exclusive
//          scan of each digit row over the blocks (one block per digit) |
//          barrier | digit bases + stable scatter of the chunk in 4096-item
//          tiles (in-warp ranks via __match_any_sync, per-warp counters) |
//          barrier.
// The item count may come from device memory (n_dev) so the pipeline needs
// no host round trip to size a sort.
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdio>

#include "primitives.cuh"

namespace hgs {

namespace cg = cooperative_groups;

namespace {

constexpr int kCoopThreads = 256;
constexpr int kItems = 16;
constexpr int kTileItems = kCoopThreads * kItems;  // 4096
constexpr int kWarps = kCoopThreads / 32;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive scan of one value per thread over a 256-thread block; also
// returns the block total.  Ends with a barrier (shared scratch reusable).
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t& total) {
    __shared__ uint32_t wt[kWarps + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t incl = warp_incl_scan(v);
    if (lane == 31) wt[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < kWarps ? wt[lane] : 0u;
        const uint32_t wi = warp_incl_scan(w);
        if (lane < kWarps) wt[lane] = wi - w;
        if (lane == kWarps - 1) wt[kWarps] = wi;
    }
    __syncthreads();
    const uint32_t ex = incl - v + wt[warp];
    total = wt[kWarps];
    __syncthreads();
    return ex;
}

__device__ __forceinline__ uint32_t block_sum(uint32_t v) {
    uint32_t t;
    block_excl_scan(v, t);
    return t;
}

__global__ void __launch_bounds__(kCoopThreads) scan_coop_kernel(const uint32_t* in, uint32_t* out, int n,
                                                                 const uint32_t* __restrict__ n_dev,
                                                                 uint32_t* __restrict__ total,
                                                                 uint32_t* __restrict__ bsum) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (coop_launch)
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    if (n_dev) n = (int)*n_dev;
    const int C = ((n + G - 1) / G + 3) & ~3;
    const int lo = min(b * C, n), hi = min(lo + C, n);
    uint32_t s = 0;
    for (int i = lo + tid; i < hi; i += kCoopThreads) s += in[i];
    s = block_sum(s);
    if (tid == 0) bsum[b] = s;
    grid.sync();
    uint32_t part = 0;
    for (int c = tid; c < b; c += kCoopThreads) part += bsum[c];
    uint32_t run = block_sum(part);
    if (b == G - 1 && tid == 0 && total) *total = run + bsum[b];
    for (int t0 = lo; t0 < hi; t0 += kTileItems) {
        const int base = t0 + tid * kItems;
        uint32_t v[kItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            v[k] = base + k < hi ? in[base + k] : 0u;
            sum += v[k];
        }
        uint32_t tot;
        uint32_t r = run + block_excl_scan(sum, tot);
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            if (base + k < hi) out[base + k] = r;
            r += v[k];
        }
        run += tot;
    }
}

// Stream compaction of the visible Gaussians (ntiles > 0) into the depth
// sort's input, in index order: keys[r] = depth_key[i], vals[r] = i, *total =
// the visible count -- the scan kernel's structure with the flag test and the
// scatter fused in (one launch instead of flag / scan / scatter).
__global__ void __launch_bounds__(kCoopThreads) compact_coop_kernel(const uint32_t* __restrict__ ntiles,
                                                                    const uint32_t* __restrict__ depth_key, int n,
                                                                    uint32_t* __restrict__ keys,
                                                                    uint32_t* __restrict__ vals,
                                                                    uint32_t* __restrict__ total,
                                                                    uint32_t* __restrict__ bsum) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (coop_launch)
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const int C = ((n + G - 1) / G + 3) & ~3;
    const int lo = min(b * C, n), hi = min(lo + C, n);
    uint32_t s = 0;
    for (int i = lo + tid; i < hi; i += kCoopThreads) s += ntiles[i] > 0u ? 1u : 0u;
    s = block_sum(s);
    if (tid == 0) bsum[b] = s;
    grid.sync();
    uint32_t part = 0;
    for (int c = tid; c < b; c += kCoopThreads) part += bsum[c];
    uint32_t run = block_sum(part);
    if (b == G - 1 && tid == 0) *total = run + bsum[b];
    for (int t0 = lo; t0 < hi; t0 += kTileItems) {
        const int base = t0 + tid * kItems;
        uint32_t v[kItems], sum = 0;
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            v[k] = base + k < hi && ntiles[base + k] > 0u ? 1u : 0u;
            sum += v[k];
        }
        uint32_t tot;
        uint32_t r = run + block_excl_scan(sum, tot);
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            if (v[k]) {
                keys[r] = depth_key[base + k];
                vals[r] = (uint32_t)(base + k);
            }
            r += v[k];
        }
        run += tot;
    }
}

struct CoopSort {
    uint32_t *k0, *v0, *k1, *v1;
    const uint32_t* n_dev;
    uint2* ranges;  // optional: [first, end) of every key's run in the sorted keys (the tile ranges)
    int n, shift0, npasses;
    uint32_t* hist;    // [256][G]
    uint32_t* rowsum;  // [256]
};

// (3 blocks/SM, 80 registers: at configs[4] sizes the passes are latency
// bound at 2 blocks/SM -- 97 registers -- and 4 (64, spilling) measured slower)
__global__ void __launch_bounds__(kCoopThreads, 3) radix_sort_coop_kernel(CoopSort a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (coop_launch)
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t h[256];
    __shared__ uint32_t cnt[kWarps][256];
    __shared__ uint32_t goff[256];
    __shared__ uint32_t dstart[256];
    __shared__ uint32_t s_k[kTileItems], s_v[kTileItems];  // the tile, stably sorted by digit
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = a.n_dev ? (int)*a.n_dev : a.n;
    HGS_DCHECK(!a.n_dev || n <= a.n);
    const int C = ((n + G - 1) / G + 31) & ~31;
    const int lo = min(b * C, n), hi = min(lo + C, n);
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t *ki = a.k0, *vi = a.v0, *ko = a.k1, *vo = a.v1;
    for (int p = 0; p < a.npasses; ++p) {
        const int shift = a.shift0 + 8 * p;
        // 1. digit histogram of this block's chunk
        h[tid] = 0u;
        __syncthreads();
        for (int i = lo + tid; i < hi; i += kCoopThreads) atomicAdd(&h[(ki[i] >> shift) & 255u], 1u);
        __syncthreads();
        a.hist[tid * G + b] = h[tid];
        grid.sync();
        // 2. exclusive scan of each digit row over the blocks
        for (int d = b; d < 256; d += G) {
            uint32_t* row = a.hist + (size_t)d * G;
            uint32_t run = 0;
            for (int c0 = 0; c0 < G; c0 += kCoopThreads) {
                const int c = c0 + tid;
                const uint32_t x = c < G ? row[c] : 0u;
                uint32_t tot;
                const uint32_t ex = block_excl_scan(x, tot);
                if (c < G) row[c] = run + ex;
                run += tot;
            }
            if (tid == 0) a.rowsum[d] = run;
        }
        grid.sync();
        // 3. global digit bases, then the stable scatter of the chunk
        {
            uint32_t tot;
            const uint32_t base = block_excl_scan(a.rowsum[tid], tot);
            goff[tid] = base + a.hist[tid * G + b];
        }
        // rounds per warp: a chunk smaller than a full 4096-item tile is spread
        // over all 8 warps (R rounds of 32 consecutive items each) instead of
        // 16 serial rounds on the first warps
        const int R = min(kItems, max(1, (hi - lo + kCoopThreads - 1) / kCoopThreads));
        for (int t0 = lo; t0 < hi; t0 += R * kCoopThreads) {
            for (int i = tid; i < kWarps * 256; i += kCoopThreads) (&cnt[0][0])[i] = 0u;
            __syncthreads();
            const int wbase = t0 + warp * (R * 32);
            uint32_t k[kItems], v[kItems], rank[kItems];
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                if (r >= R) break;
                const int idx = wbase + r * 32 + lane;
                const bool valid = idx < hi;
                k[r] = valid ? ki[idx] : 0u;
                v[r] = valid ? vi[idx] : 0u;
                const uint32_t d = valid ? ((k[r] >> shift) & 255u) : 256u;
                const unsigned peers = __match_any_sync(0xffffffffu, d);
                const uint32_t before = valid ? cnt[warp][d] : 0u;
                __syncwarp();
                if (valid && lane == __ffs(peers) - 1) cnt[warp][d] = before + __popc(peers);
                __syncwarp();
                rank[r] = before + __popc(peers & lt_mask);
            }
            __syncthreads();
            uint32_t tile_tot = 0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t t = cnt[w][tid];
                cnt[w][tid] = tile_tot;
                tile_tot += t;
            }
            {
                uint32_t all;
                dstart[tid] = block_excl_scan(tile_tot, all);
            }
            __syncthreads();
            // the tile, stably sorted by digit, in shared memory ...
#pragma unroll
            for (int r = 0; r < kItems; ++r) {
                if (r >= R) break;
                const int idx = wbase + r * 32 + lane;
                if (idx < hi) {
                    const uint32_t d = (k[r] >> shift) & 255u;
                    const uint32_t lp = dstart[d] + cnt[warp][d] + rank[r];
                    s_k[lp] = k[r];
                    s_v[lp] = v[r];
                }
            }
            __syncthreads();
            // ... written out in order: consecutive threads write consecutive
            // addresses of each digit's run (coalesced)
            const int nt = min(R * kCoopThreads, hi - t0);
            for (int q = tid; q < nt; q += kCoopThreads) {
                const uint32_t kk = s_k[q];
                const uint32_t d = (kk >> shift) & 255u;
                const uint32_t pos = goff[d] + (uint32_t)q - dstart[d];
                HGS_DCHECK(pos < (uint32_t)n);
                ko[pos] = kk;
                vo[pos] = s_v[q];
            }
            __syncthreads();
            goff[tid] += tile_tot;
        }
        grid.sync();
        uint32_t* t = ki;
        ki = ko;
        ko = t;
        t = vi;
        vi = vo;
        vo = t;
    }
    if (a.ranges) {  // run boundaries of the sorted keys (after the last barrier)
        for (int i = lo + tid; i < hi; i += kCoopThreads) {
            const uint32_t t = ki[i];
            if (i == 0 || ki[i - 1] != t) a.ranges[t].x = (uint32_t)i;
            if (i == n - 1 || ki[i + 1] != t) a.ranges[t].y = (uint32_t)(i + 1);
        }
    }
}

// Grid of a cooperative kernel for n items: co-resident (<= 4 blocks per SM
// and the occupancy limit), at least one block per SM, about 2048 items per
// block -- small sorts pay for fewer blocks at every grid barrier.
template <typename K>
int coop_grid(K kernel, int n) {
    static int cached[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cached[dev][0]) {
        int per_sm = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kCoopThreads, 0);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cached[dev][0] = std::max(1, std::min(per_sm, 4)) * sms;
        cached[dev][1] = sms;
    }
    const int want = std::max(cached[dev][1], (int)div_up((uint32_t)std::max(n, 1), 2048u));
    return std::min(cached[dev][0], want);
}

constexpr int kMaxCoopGrid = 4 * 256;  // workspace bound (<= 4 blocks/SM on <= 256 SMs)

}  // namespace

size_t scan_workspace_bytes(int) { return (size_t)(kMaxCoopGrid + 32) * sizeof(uint32_t); }

bool pdl_enabled();  // capi.cu

// Cooperative launch (grid-wide barriers) that may also be scheduled while
// its predecessor drains (programmatic dependent launch; the kernels start
// with griddepcontrol.wait).
cudaError_t coop_launch(const void* kernel, int grid, void** args, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCoopThreads);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelExC(&cfg, kernel, args);
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, int n, uint32_t* total, uint32_t* ws, cudaStream_t st,
                        const uint32_t* n_dev) {
    if (n <= 0 && !n_dev) {
        if (total) cudaMemsetAsync(total, 0, sizeof(uint32_t), st);
        return;
    }
    const int G = std::min(coop_grid(scan_coop_kernel, n), kMaxCoopGrid);
    void* args[] = {(void*)&in, (void*)&out, (void*)&n, (void*)&n_dev, (void*)&total, (void*)&ws};
    coop_launch((const void*)scan_coop_kernel, G, args, st);
    count_launch();
}

void compact_visible(const uint32_t* ntiles, const uint32_t* depth_key, int n, uint32_t* keys, uint32_t* vals,
                     uint32_t* total, uint32_t* ws, cudaStream_t st) {
    if (n <= 0) {
        cudaMemsetAsync(total, 0, sizeof(uint32_t), st);
        return;
    }
    const int G = std::min(coop_grid(compact_coop_kernel, n), kMaxCoopGrid);
    void* args[] = {(void*)&ntiles, (void*)&depth_key, (void*)&n, (void*)&keys, (void*)&vals, (void*)&total, (void*)&ws};
    coop_launch((const void*)compact_coop_kernel, G, args, st);
    count_launch();
}

size_t radix_workspace_bytes(int) { return (size_t)(256 * kMaxCoopGrid + 256 + 64) * sizeof(uint32_t); }

// Stable LSD sort of (keys, vals) on bits [begin_bit, end_bit).  The result
// lands in (keys, vals) when the pass count is even, else in (keys_alt,
// vals_alt); the return value says which (0 = original buffers).
int radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_alt, uint32_t* vals_alt, int n,
                     int begin_bit, int end_bit, uint32_t* ws, cudaStream_t st, const uint32_t* n_dev,
                     uint2* ranges) {
    if (!n_dev && n <= 1) return 0;
    const int npasses = (end_bit - begin_bit + 7) / 8;
    if (npasses <= 0) return 0;
    CoopSort a;
    a.k0 = keys;
    a.v0 = vals;
    a.k1 = keys_alt;
    a.v1 = vals_alt;
    a.n_dev = n_dev;
    a.ranges = ranges;
    a.n = n;
    a.shift0 = begin_bit;
    a.npasses = npasses;
    a.hist = ws;
    a.rowsum = ws + 256 * kMaxCoopGrid;
    const int G = std::min(coop_grid(radix_sort_coop_kernel, n), kMaxCoopGrid);
    void* args[] = {(void*)&a};
    coop_launch((const void*)radix_sort_coop_kernel, G, args, st);
    count_launch();
    return npasses & 1;
}

}  // namespace hgs

#include <atomic>
namespace hgs {
static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
}  // namespace hgs
