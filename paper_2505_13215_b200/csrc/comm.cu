// comm.cu -- the multi-GPU exchange of SURVEY.md 8e behind the C ABI.
//
// View-parallel data parallelism: every rank holds a replica of the scene and
// renders its share of the batch; the one exchange per optimizer step is an
// all-reduce (sum) of the valid gradient rows + densify-statistic deltas,
// in place (one NCCL group), then every rank applies the same Adam step.  Replica consistency is checked with an order-independent
// 64-bit checksum of the parameters (hgs_param_checksum) and repaired with a
// broadcast from a root (hgs_broadcast_params).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): a process that
// already loaded torch's NCCL shares that copy, a plain C++ caller gets the
// system one; nothing links NCCL into libhgs_gpu.so.
#include <dlfcn.h>
#include <link.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <initializer_list>
#include <utility>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

struct NcclApi {
    bool loaded = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    std::string path;  // the library the symbols came from
};

// The NCCL already mapped into the process (e.g. torch's bundled copy), so a
// process holds one NCCL; else the first libnccl.so.2 on the search path.
int find_loaded_nccl(struct dl_phdr_info* info, size_t, void* out) {
    const char* n = info->dlpi_name;
    if (n && std::strstr(n, "libnccl.so")) {
        *static_cast<std::string*>(out) = n;
        return 1;
    }
    return 0;
}

// ---- loopback collectives (HGS_NCCL_LOOPBACK=1): the NCCL entry points
// replaced by an in-process implementation for ranks that are threads of one
// process sharing one device -- the test double that runs the N > 1 exchange
// (all-reduce, reduce-scatter, all-gather, broadcast: every collective this
// file issues) on a single GPU, where NCCL refuses two ranks per device.
// Each call is a host barrier over the group; the last rank to arrive makes
// its stream wait for every rank's inputs, combines them in rank order into
// a scratch buffer (so in-place calls read before anything is written),
// copies each rank's result out and records an event every rank's stream
// waits on.  Group calls are executed one by one (every rank issues the same
// sequence).
enum LoopKind { LK_ALLREDUCE, LK_REDUCE_SCATTER, LK_ALLGATHER, LK_BROADCAST };
constexpr int kLoopMaxRanks = 8;

struct LoopCall {
    const void* send;
    void* recv;
    cudaStream_t st;
};
struct LoopGroup {
    int world = 0, joined = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    LoopCall calls[kLoopMaxRanks];
    cudaEvent_t ready[kLoopMaxRanks] = {};
    cudaEvent_t done = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
};
struct LoopRank {
    LoopGroup* g;
    int rank;
};
std::mutex g_loop_mu;
std::map<unsigned long long, LoopGroup*> g_loop_groups;
unsigned long long g_loop_next = 1;

struct LoopSrc {
    const void* p[kLoopMaxRanks];
};

template <typename T>
__global__ void loop_combine_kernel(LoopSrc src, int world, int kind, int root, size_t count, T* __restrict__ out) {
    const size_t total = (kind == LK_ALLREDUCE || kind == LK_BROADCAST) ? count : count * (size_t)world;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        T v;
        if (kind == LK_ALLGATHER) {
            v = static_cast<const T*>(src.p[i / count])[i % count];
        } else if (kind == LK_BROADCAST) {
            v = static_cast<const T*>(src.p[root])[i];
        } else {
            v = static_cast<const T*>(src.p[0])[i];
            for (int k = 1; k < world; ++k) v += static_cast<const T*>(src.p[k])[i];
        }
        out[i] = v;
    }
}

size_t loop_type_size(ncclDataType_t t) {
    return (t == ncclFloat64 || t == ncclUint64 || t == ncclInt64) ? 8 : 4;
}

ncclResult_t loop_collective(int kind, const void* send, void* recv, size_t count, ncclDataType_t type, int root,
                             ncclComm_t comm, cudaStream_t st) {
    LoopRank* me = reinterpret_cast<LoopRank*>(comm);
    LoopGroup& g = *me->g;
    if (cudaEventRecord(g.ready[me->rank], st) != cudaSuccess) return ncclUnhandledCudaError;
    std::unique_lock<std::mutex> lk(g.mu);
    g.calls[me->rank] = LoopCall{send, recv, st};
    const unsigned long long gen = g.gen;
    if (++g.arrived < g.world) {
        g.cv.wait(lk, [&] { return g.gen != gen; });
    } else {
        const size_t es = loop_type_size(type);
        const size_t total = (kind == LK_ALLREDUCE || kind == LK_BROADCAST) ? count : count * (size_t)g.world;
        bool ok = true;
        for (int k = 0; k < g.world; ++k) ok &= cudaStreamWaitEvent(st, g.ready[k], 0) == cudaSuccess;
        if (total * es > g.tmp_bytes) {
            ok &= cudaStreamSynchronize(st) == cudaSuccess;
            if (g.tmp) cudaFree(g.tmp);
            g.tmp = nullptr;
            ok &= cudaMalloc(&g.tmp, total * es) == cudaSuccess;
            g.tmp_bytes = ok ? total * es : 0;
        }
        if (ok && total > 0) {
            LoopSrc src{};
            for (int k = 0; k < g.world; ++k) src.p[k] = g.calls[k].send;
            const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, 4096);
            if (type == ncclFloat32)
                loop_combine_kernel<float><<<blocks, 256, 0, st>>>(src, g.world, kind, root, count,
                                                                   static_cast<float*>(g.tmp));
            else if (type == ncclFloat64)
                loop_combine_kernel<double><<<blocks, 256, 0, st>>>(src, g.world, kind, root, count,
                                                                    static_cast<double*>(g.tmp));
            else if (es == 8)
                loop_combine_kernel<unsigned long long><<<blocks, 256, 0, st>>>(
                    src, g.world, kind, root, count, static_cast<unsigned long long*>(g.tmp));
            else
                loop_combine_kernel<uint32_t><<<blocks, 256, 0, st>>>(src, g.world, kind, root, count,
                                                                      static_cast<uint32_t*>(g.tmp));
            for (int k = 0; k < g.world; ++k) {
                const char* from = static_cast<const char*>(g.tmp);
                size_t n = count * es;
                if (kind == LK_REDUCE_SCATTER) from += (size_t)k * count * es;
                if (kind == LK_ALLGATHER) n = total * es;
                ok &= cudaMemcpyAsync(g.calls[k].recv, from, n, cudaMemcpyDeviceToDevice, st) == cudaSuccess;
            }
        }
        ok &= cudaEventRecord(g.done, st) == cudaSuccess;
        g.arrived = 0;
        ++g.gen;
        g.cv.notify_all();
        if (!ok) return ncclUnhandledCudaError;
    }
    lk.unlock();
    return cudaStreamWaitEvent(st, g.done, 0) == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t loop_get_unique_id(ncclUniqueId* id) {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    std::memset(id, 0, sizeof(*id));
    const unsigned long long key = g_loop_next++;
    std::memcpy(id->internal, &key, sizeof(key));
    return ncclSuccess;
}
ncclResult_t loop_comm_init_rank(ncclComm_t* comm, int world, ncclUniqueId id, int rank) {
    if (world < 1 || world > kLoopMaxRanks || rank < 0 || rank >= world) return ncclInvalidArgument;
    unsigned long long key;
    std::memcpy(&key, id.internal, sizeof(key));
    std::lock_guard<std::mutex> lk(g_loop_mu);
    LoopGroup*& g = g_loop_groups[key];
    if (!g) {
        g = new LoopGroup();
        g->world = world;
        for (int k = 0; k < world; ++k) cudaEventCreateWithFlags(&g->ready[k], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming);
    }
    if (g->world != world) return ncclInvalidArgument;
    ++g->joined;
    *comm = reinterpret_cast<ncclComm_t>(new LoopRank{g, rank});
    return ncclSuccess;
}
ncclResult_t loop_comm_init_all(ncclComm_t*, int, const int*) { return ncclInvalidUsage; }
ncclResult_t loop_comm_destroy(ncclComm_t comm) {
    LoopRank* me = reinterpret_cast<LoopRank*>(comm);
    std::lock_guard<std::mutex> lk(g_loop_mu);
    delete me;  // (the group stays: its events may still be waited on)
    return ncclSuccess;
}
ncclResult_t loop_all_reduce(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t, ncclComm_t c,
                             cudaStream_t st) {
    return loop_collective(LK_ALLREDUCE, s, r, n, t, 0, c, st);
}
ncclResult_t loop_broadcast(const void* s, void* r, size_t n, ncclDataType_t t, int root, ncclComm_t c,
                            cudaStream_t st) {
    return loop_collective(LK_BROADCAST, s, r, n, t, root, c, st);
}
ncclResult_t loop_reduce_scatter(const void* s, void* r, size_t n, ncclDataType_t t, ncclRedOp_t, ncclComm_t c,
                                 cudaStream_t st) {
    return loop_collective(LK_REDUCE_SCATTER, s, r, n, t, 0, c, st);
}
ncclResult_t loop_all_gather(const void* s, void* r, size_t n, ncclDataType_t t, ncclComm_t c, cudaStream_t st) {
    return loop_collective(LK_ALLGATHER, s, r, n, t, 0, c, st);
}
ncclResult_t loop_group() { return ncclSuccess; }
const char* loop_error_string(ncclResult_t r) { return r == ncclSuccess ? "success" : "loopback collective failed"; }
ncclResult_t loop_version(int* v) {
    *v = 0;
    return ncclSuccess;
}

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        if (getenv("HGS_NCCL_LOOPBACK")) {  // in-process test double (above)
            a.GetUniqueId = loop_get_unique_id;
            a.CommInitRank = loop_comm_init_rank;
            a.CommInitAll = loop_comm_init_all;
            a.CommDestroy = loop_comm_destroy;
            a.AllReduce = loop_all_reduce;
            a.Broadcast = loop_broadcast;
            a.ReduceScatter = loop_reduce_scatter;
            a.AllGather = loop_all_gather;
            a.GroupStart = loop_group;
            a.GroupEnd = loop_group;
            a.GetErrorString = loop_error_string;
            a.GetVersion = loop_version;
            a.path = "loopback";
            a.loaded = true;
            return a;
        }
        std::string loaded;
        dl_iterate_phdr(find_loaded_nccl, &loaded);
        void* h = loaded.empty() ? nullptr : dlopen(loaded.c_str(), RTLD_NOW | RTLD_NOLOAD);
        a.path = loaded;
        if (!h) {
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            a.path = "libnccl.so.2";
        }
        if (!h) {
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            a.path = "libnccl.so";
        }
        if (!h) {
            a.err = std::string("NCCL not found: ") + dlerror();
            return a;
        }
#define SYM(f)                                                             \
    a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f));            \
    if (!a.f) {                                                            \
        a.err = "NCCL symbol missing: nccl" #f;                            \
        return a;                                                          \
    }
        SYM(GetUniqueId) SYM(CommInitRank) SYM(CommInitAll) SYM(CommDestroy) SYM(AllReduce) SYM(Broadcast)
        SYM(ReduceScatter) SYM(AllGather) SYM(GroupStart) SYM(GroupEnd) SYM(GetErrorString) SYM(GetVersion)
#undef SYM
        a.loaded = true;
        return a;
    }();
    return api;
}

hgs_status fail(hgs_ctx* ctx, hgs_status s, const std::string& m) {
    if (ctx) ctx->err = m;
    return s;
}

#define CKC(x)                                                                                    \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) return fail(ctx, HGS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define CKN(x)                                                                                            \
    do {                                                                                                  \
        ncclResult_t r_ = (x);                                                                            \
        if (r_ != ncclSuccess) return fail(ctx, HGS_ERR_CUDA, std::string("NCCL: ") + nccl().GetErrorString(r_)); \
    } while (0)

hgs_status need_nccl(hgs_ctx* ctx) {
    if (!nccl().loaded) return fail(ctx, HGS_ERR_CUDA, nccl().err);
    return HGS_OK;
}

hgs_status need_comm(hgs_ctx* ctx) {
    if (!ctx->comm) return fail(ctx, HGS_ERR_STATE, "comm: call hgs_comm_init / hgs_comm_init_all first");
    return HGS_OK;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {  // splitmix64 finaliser
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// order-independent checksum: sum over valid elements of mix64(bits, position)
__global__ void checksum_kernel(const float* __restrict__ p, int64_t cap, int64_t n, int rows, unsigned long long salt,
                                unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    const int64_t total = n * rows;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / n, i = e - r * n;
        const unsigned long long bits = __float_as_uint(p[r * cap + i]);
        acc += mix64(bits ^ ((unsigned long long)e << 32) ^ salt);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Zero rows [0, span) of `rows` rows (stride cap) outside [lo, hi): the
// gradient entries a reduce-scatter left unreduced on this rank.
__global__ void zero_outside_kernel(float* __restrict__ base, int64_t cap, int rows, int64_t span, int64_t lo,
                                    int64_t hi) {
    const int64_t total = span * rows;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / span, i = e - r * span;
        if (i < lo || i >= hi) base[r * cap + i] = 0.0f;
    }
}

__global__ void add_u64_kernel(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src) {
    *dst += *src;
}

int64_t shard_chunk(int64_t n, int ranks) { return ranks > 0 ? ((n + ranks - 1) / ranks + 3) / 4 * 4 : n; }

}  // namespace

hgs_status comm_allreduce_f64_dev(hgs_ctx* ctx, double* dev, int n) {
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    if (n > 0)
        CKN(nccl().AllReduce(dev, dev, (size_t)n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx->comm),
                             ctx->stream));
    return HGS_OK;
}

// Every row of the pools (and the statistic rows) of n Gaussians, chunk c
// per rank: the in-place collectives need ranks * c <= capacity, which
// round_cap (n rounded up to 128, + 128) guarantees for <= 32 ranks.
hgs_status comm_check_chunks(hgs_ctx* ctx, int64_t& c4, int64_t& c3) {
    c4 = shard_chunk(ctx->n4, ctx->comm_size);
    c3 = shard_chunk(ctx->n3, ctx->comm_size);
    if (c4 * ctx->comm_size > ctx->cap4 || c3 * ctx->comm_size > ctx->cap3)
        return fail(ctx, HGS_ERR_STATE, "sharded exchange: pool capacity below ranks x chunk");
    return HGS_OK;
}

// Reduce-scatter of every gradient row and statistic-delta row: rank r
// receives the sum of [r c, r c + c) in place.
hgs_status comm_reduce_scatter_grads(hgs_ctx* ctx) {
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    int64_t c4, c3;
    r = comm_check_chunks(ctx, c4, c3);
    if (r != HGS_OK) return r;
    ncclComm_t c = static_cast<ncclComm_t>(ctx->comm);
    const int rk = ctx->comm_rank;
    auto rs = [&](float* row, int64_t ch) -> ncclResult_t {
        return ch > 0 ? nccl().ReduceScatter(row, row + (int64_t)rk * ch, (size_t)ch, ncclFloat32, ncclSum, c,
                                             ctx->stream)
                      : ncclSuccess;
    };
    ctx->grads_zero = false;
    CKN(nccl().GroupStart());
    for (int k = 0; k < rows4(ctx->deg); ++k) CKN(rs(ctx->g4 + (int64_t)k * ctx->cap4, c4));
    for (int k = 0; k < rows3(ctx->deg); ++k) CKN(rs(ctx->g3 + (int64_t)k * ctx->cap3, c3));
    CKN(rs(ctx->dgn4, c4));
    CKN(rs(ctx->dcnt4, c4));
    CKN(rs(ctx->dgn3, c3));
    CKN(rs(ctx->dcnt3, c3));
    CKN(nccl().GroupEnd());
    return HGS_OK;
}

// All-gather of row sets: rank r contributes [r c, r c + c) of every row.
hgs_status comm_allgather_rows(hgs_ctx* ctx, std::initializer_list<std::pair<float*, int>> sets4,
                               std::initializer_list<std::pair<float*, int>> sets3) {
    int64_t c4, c3;
    hgs_status r = comm_check_chunks(ctx, c4, c3);
    if (r != HGS_OK) return r;
    ncclComm_t c = static_cast<ncclComm_t>(ctx->comm);
    const int rk = ctx->comm_rank;
    auto ag = [&](float* row, int64_t ch) -> ncclResult_t {
        return ch > 0 ? nccl().AllGather(row + (int64_t)rk * ch, row, (size_t)ch, ncclFloat32, c, ctx->stream)
                      : ncclSuccess;
    };
    CKN(nccl().GroupStart());
    for (const auto& s : sets4)
        for (int k = 0; k < s.second; ++k) CKN(ag(s.first + (int64_t)k * ctx->cap4, c4));
    for (const auto& s : sets3)
        for (int k = 0; k < s.second; ++k) CKN(ag(s.first + (int64_t)k * ctx->cap3, c3));
    CKN(nccl().GroupEnd());
    return HGS_OK;
}

// After the sharded Adam: this rank's gradients outside its shard were
// never reduced (zeroed here; the shard itself was zeroed by Adam), the
// updated parameters and folded statistics are all-gathered, and the step's
// skipped-class count is summed over the ranks into skipped_nonfinite.
hgs_status comm_sharded_finish(hgs_ctx* ctx, unsigned long long* skipped, unsigned long long* skipped_cum) {
    int64_t c4, c3;
    hgs_status r = comm_check_chunks(ctx, c4, c3);
    if (r != HGS_OK) return r;
    int64_t lo4, hi4, lo3, hi3;
    hgs_shard_range(ctx->n4, ctx->comm_size, ctx->comm_rank, &lo4, &hi4);
    hgs_shard_range(ctx->n3, ctx->comm_size, ctx->comm_rank, &lo3, &hi3);
    const int blocks = ctx->sms * 4;
    const int64_t s4 = c4 * ctx->comm_size, s3 = c3 * ctx->comm_size;
    if (s4 > 0) {
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->g4, ctx->cap4, rows4(ctx->deg), s4, lo4, hi4);
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->dgn4, ctx->cap4, 1, s4, lo4, hi4);
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->dcnt4, ctx->cap4, 1, s4, lo4, hi4);
        count_launch(3);
    }
    if (s3 > 0) {
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->g3, ctx->cap3, rows3(ctx->deg), s3, lo3, hi3);
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->dgn3, ctx->cap3, 1, s3, lo3, hi3);
        zero_outside_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->dcnt3, ctx->cap3, 1, s3, lo3, hi3);
        count_launch(3);
    }
    CKC(cudaGetLastError());
    r = comm_allgather_rows(ctx, {{ctx->p4.as<float>(), rows4(ctx->deg)}, {ctx->gn4.as<float>(), 1}, {ctx->cnt4.as<float>(), 1}},
                            {{ctx->p3.as<float>(), rows3(ctx->deg)}, {ctx->gn3.as<float>(), 1}, {ctx->cnt3.as<float>(), 1}});
    if (r != HGS_OK) return r;
    CKN(nccl().AllReduce(skipped, skipped, 1, ncclUint64, ncclSum, static_cast<ncclComm_t>(ctx->comm), ctx->stream));
    add_u64_kernel<<<1, 1, 0, ctx->stream>>>(skipped_cum, skipped);
    count_launch();
    CKC(cudaGetLastError());
    ctx->grads_zero = true;
    ctx->state_sharded = true;
    return HGS_OK;
}

extern "C" {

hgs_status hgs_comm_unique_id(hgs_comm_id* out) {
    if (!out) return HGS_ERR_INVALID_ARGUMENT;
    if (!nccl().loaded) return HGS_ERR_CUDA;
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) return HGS_ERR_CUDA;
    static_assert(sizeof(id.internal) == sizeof(out->internal), "hgs_comm_id size");
    std::memcpy(out->internal, id.internal, sizeof(id.internal));
    return HGS_OK;
}

hgs_status hgs_comm_init(hgs_ctx* ctx, int nranks, int rank, const hgs_comm_id* id) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = need_nccl(ctx);
    if (r != HGS_OK) return r;
    if (ctx->comm) return fail(ctx, HGS_ERR_STATE, "comm: already initialised");
    CKC(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    std::memcpy(uid.internal, id->internal, sizeof(uid.internal));
    ncclComm_t c = nullptr;
    CKN(nccl().CommInitRank(&c, nranks, uid, rank));
    ctx->comm = c;
    ctx->comm_rank = rank;
    ctx->comm_size = nranks;
    return HGS_OK;
}

hgs_status hgs_comm_init_all(hgs_ctx* const* ctxs, int n) {
    if (!ctxs || n < 1) return HGS_ERR_INVALID_ARGUMENT;
    hgs_ctx* ctx = ctxs[0];
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = need_nccl(ctx);
    if (r != HGS_OK) return r;
    std::vector<int> devs((size_t)n);
    for (int i = 0; i < n; ++i) {
        if (!ctxs[i]) return HGS_ERR_INVALID_ARGUMENT;
        if (ctxs[i]->comm) return fail(ctx, HGS_ERR_STATE, "comm: already initialised");
        devs[(size_t)i] = ctxs[i]->device;
    }
    std::vector<ncclComm_t> comms((size_t)n);
    CKN(nccl().CommInitAll(comms.data(), n, devs.data()));
    for (int i = 0; i < n; ++i) {
        ctxs[i]->comm = comms[(size_t)i];
        ctxs[i]->comm_rank = i;
        ctxs[i]->comm_size = n;
    }
    return HGS_OK;
}

hgs_status hgs_comm_destroy(hgs_ctx* ctx) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (ctx->comm && nccl().loaded) {
        cudaSetDevice(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    }
    ctx->comm = nullptr;
    ctx->comm_rank = 0;
    ctx->comm_size = 1;
    return HGS_OK;
}

// In place, no packing: one NCCL group of sum all-reduces over the valid
// prefix [0, n) of every gradient row (the rows are strided by the pool
// capacity, whose tail is padding) and of the densification-statistic
// deltas.  NCCL runs the group as one aggregated launch (with a one-rank
// communicator: the identity, still issued through NCCL).
hgs_status hgs_allreduce_grads(hgs_ctx* ctx) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    if (!ctx->gbuf.p) return fail(ctx, HGS_ERR_STATE, "allreduce_grads: no scene uploaded");
    CKC(cudaSetDevice(ctx->device));
    ctx->grads_zero = false;
    ncclComm_t c = static_cast<ncclComm_t>(ctx->comm);
    const int r4 = rows4(ctx->deg), r3 = rows3(ctx->deg);
    auto ar = [&](float* p, int64_t n) -> ncclResult_t {
        return n > 0 ? nccl().AllReduce(p, p, (size_t)n, ncclFloat32, ncclSum, c, ctx->stream) : ncclSuccess;
    };
    CKN(nccl().GroupStart());
    for (int k = 0; k < r4; ++k) CKN(ar(ctx->g4 + (int64_t)k * ctx->cap4, ctx->n4));
    for (int k = 0; k < r3; ++k) CKN(ar(ctx->g3 + (int64_t)k * ctx->cap3, ctx->n3));
    CKN(ar(ctx->dgn4, ctx->n4));
    CKN(ar(ctx->dgn3, ctx->n3));
    CKN(ar(ctx->dcnt4, ctx->n4));
    CKN(ar(ctx->dcnt3, ctx->n3));
    CKN(nccl().GroupEnd());
    return HGS_OK;
}

void hgs_shard_range(int64_t n, int ranks, int rank, int64_t* lo, int64_t* hi) {
    const int64_t c = shard_chunk(n, ranks);
    const int64_t l = std::min<int64_t>(n, (int64_t)rank * c);
    if (lo) *lo = l;
    if (hi) *hi = std::min<int64_t>(n, l + c);
}

hgs_status hgs_comm_set_sharded(hgs_ctx* ctx, int enable) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (enable && ctx->comm_size > 32) return fail(ctx, HGS_ERR_INVALID_ARGUMENT, "sharded exchange: at most 32 ranks");
    ctx->sharded = enable != 0;
    return HGS_OK;
}

hgs_status hgs_gather_state(hgs_ctx* ctx) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    if (!ctx->state_sharded) return HGS_OK;
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    CKC(cudaSetDevice(ctx->device));
    r = comm_allgather_rows(ctx, {{ctx->m4.as<float>(), rows4(ctx->deg)}, {ctx->v4.as<float>(), rows4(ctx->deg)}},
                            {{ctx->m3.as<float>(), rows3(ctx->deg)}, {ctx->v3.as<float>(), rows3(ctx->deg)}});
    if (r != HGS_OK) return r;
    CKC(cudaStreamSynchronize(ctx->stream));
    ctx->state_sharded = false;
    return HGS_OK;
}

hgs_status hgs_allreduce_f64(hgs_ctx* ctx, double* vals, int n) {
    if (!ctx || (n > 0 && !vals) || n < 0) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    if (n == 0) return HGS_OK;
    CKC(cudaSetDevice(ctx->device));
    CKC(ctx->comm_buf.ensure((size_t)n * 8));
    CKC(cudaMemcpyAsync(ctx->comm_buf.p, vals, (size_t)n * 8, cudaMemcpyHostToDevice, ctx->stream));
    CKN(nccl().AllReduce(ctx->comm_buf.p, ctx->comm_buf.p, (size_t)n, ncclFloat64, ncclSum,
                         static_cast<ncclComm_t>(ctx->comm), ctx->stream));
    CKC(cudaMemcpyAsync(vals, ctx->comm_buf.p, (size_t)n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

hgs_status hgs_param_checksum(hgs_ctx* ctx, uint64_t* out) {
    if (!ctx || !out) return HGS_ERR_INVALID_ARGUMENT;
    CKC(cudaSetDevice(ctx->device));
    CKC(ctx->comm_buf.ensure(64));
    unsigned long long* d = ctx->comm_buf.as<unsigned long long>();
    CKC(cudaMemsetAsync(d, 0, 8, ctx->stream));
    const int blocks = ctx->sms * 4;
    if (ctx->n4)
        checksum_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->p4.as<float>(), ctx->cap4, ctx->n4, rows4(ctx->deg),
                                                         0x4444ull, d);
    if (ctx->n3)
        checksum_kernel<<<blocks, 256, 0, ctx->stream>>>(ctx->p3.as<float>(), ctx->cap3, ctx->n3, rows3(ctx->deg),
                                                         0x3333ull << 40, d);
    count_launch((ctx->n4 ? 1 : 0) + (ctx->n3 ? 1 : 0));
    CKC(cudaGetLastError());
    unsigned long long h = 0;
    CKC(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    *out = (uint64_t)(h ^ ((uint64_t)ctx->n4 << 1) ^ ((uint64_t)ctx->n3 << 33));
    return HGS_OK;
}

hgs_status hgs_broadcast_params(hgs_ctx* ctx, int root) {
    if (!ctx) return HGS_ERR_INVALID_ARGUMENT;
    hgs_status r = need_comm(ctx);
    if (r != HGS_OK) return r;
    r = hgs_gather_state(ctx);  // the moments whole on every rank before root's are broadcast
    if (r != HGS_OK) return r;
    if (root < 0 || root >= ctx->comm_size) return HGS_ERR_INVALID_ARGUMENT;
    CKC(cudaSetDevice(ctx->device));
    // every rank must hold the same pool sizes (the replicas diverged in
    // values, not in structure)
    const size_t b4 = (size_t)rows4(ctx->deg) * ctx->cap4, b3 = (size_t)rows3(ctx->deg) * ctx->cap3;
    ncclComm_t c = static_cast<ncclComm_t>(ctx->comm);
    CKN(nccl().GroupStart());
    for (DBuf* b : {&ctx->p4, &ctx->m4, &ctx->v4})
        CKN(nccl().Broadcast(b->p, b->p, b4, ncclFloat32, root, c, ctx->stream));
    for (DBuf* b : {&ctx->p3, &ctx->m3, &ctx->v3})
        CKN(nccl().Broadcast(b->p, b->p, b3, ncclFloat32, root, c, ctx->stream));
    for (DBuf* b : {&ctx->gn4, &ctx->cnt4})
        CKN(nccl().Broadcast(b->p, b->p, (size_t)ctx->cap4, ncclFloat32, root, c, ctx->stream));
    for (DBuf* b : {&ctx->gn3, &ctx->cnt3})
        CKN(nccl().Broadcast(b->p, b->p, (size_t)ctx->cap3, ncclFloat32, root, c, ctx->stream));
    CKN(nccl().GroupEnd());
    CKC(cudaStreamSynchronize(ctx->stream));
    return HGS_OK;
}

// The NCCL the exchange uses: its version code (ncclGetVersion) and path.
hgs_status hgs_comm_nccl_info(int* version, char* path, int path_len) {
    if (!nccl().loaded) return HGS_ERR_CUDA;
    if (version && nccl().GetVersion(version) != ncclSuccess) return HGS_ERR_CUDA;
    if (path && path_len > 0) {
        std::strncpy(path, nccl().path.c_str(), (size_t)path_len - 1);
        path[path_len - 1] = 0;
    }
    return HGS_OK;
}

int hgs_comm_size(hgs_ctx* ctx) { return ctx ? ctx->comm_size : 0; }
int hgs_comm_rank(hgs_ctx* ctx) { return ctx ? ctx->comm_rank : 0; }

}  // extern "C"
