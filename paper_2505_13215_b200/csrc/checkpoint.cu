// checkpoint.cu -- versioned, CRC-32-checked .hgsc checkpoints
// (data_io.cpp:444-719), byte-compatible with the reference.
//
// Device scenes: the record / array payloads are produced and consumed by
// CUDA kernels directly from / into the FP32 SoA pools -- one CTA per 32
// Gaussians stages the rows in shared memory and writes (reads) the
// Gaussian-major byte stream coalesced; the host adds the ~40 header scalars,
// computes the CRC-32 (zlib, as the reference) and moves the bytes.
//
// The SoA row order of both pools equals the field order of a checkpoint
// record (hgs_common.cuh R3_* / R4_*): a record is rows [0, pre) as f64, the
// u32 SH degree, rows [pre, rows) as f64 (pre = R3_SH / R4_SH).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "train_api.cuh"

using namespace hgs;

namespace {

constexpr uint32_t kVersion = 1;  // data_io.cpp:448
constexpr int kMaxDeg = 3;
constexpr uint64_t kScenHdr = 44;  // u32 deg, f64 tau, duration, extent, u64 n3, n4
constexpr int kTileG = 32;          // Gaussians per CTA
constexpr int kPad = kTileG + 1;    // padded shared-memory row (bank-conflict free transposes)
constexpr uint32_t CKPT_BAD_DEG = 1u, CKPT_NONUNIT = 2u;

thread_local std::string g_io_err;

struct IoError {
    hgs_status code = HGS_OK;
    std::string msg;
};

#define CKC(x)                                                                                       \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess) {                                                                     \
            ctx->err = std::string(#x) + ": " + cudaGetErrorString(e_);                              \
            return HGS_ERR_CUDA;                                                                     \
        }                                                                                            \
    } while (0)
#define CKL()                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = cudaGetLastError();                                                         \
        if (e_ != cudaSuccess) {                                                                     \
            ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e_);                      \
            return HGS_ERR_CUDA;                                                                     \
        }                                                                                            \
    } while (0)

// ------------------------------------------------------------------ kernels

// SoA rows of n Gaussians -> checkpoint records (rows*2+1 u32 words each)
__global__ void __launch_bounds__(256) encode_records_kernel(const float* __restrict__ src, int64_t cap, int64_t n,
                                                             int rows, int pre, uint32_t deg,
                                                             uint32_t* __restrict__ out) {
    extern __shared__ float tile[];  // [rows][kPad]
    const int64_t base = (int64_t)blockIdx.x * kTileG;
    const int cnt = (int)(n - base < kTileG ? n - base : (int64_t)kTileG);
    for (int i = threadIdx.x; i < rows * kTileG; i += blockDim.x) {
        const int k = i >> 5, g = i & 31;
        tile[k * kPad + g] = g < cnt ? src[(int64_t)k * cap + base + g] : 0.f;
    }
    __syncthreads();
    const int wpr = 2 * rows + 1;
    uint32_t* o = out + base * wpr;
    for (int w = threadIdx.x; w < cnt * wpr; w += blockDim.x) {
        const int r = w / wpr, q = w - r * wpr;
        uint32_t v;
        if (q == 2 * pre) {
            v = deg;
        } else {
            const int qq = q < 2 * pre ? q : q - 1;
            const unsigned long long b = (unsigned long long)__double_as_longlong((double)tile[(qq >> 1) * kPad + r]);
            v = (qq & 1) ? (uint32_t)(b >> 32) : (uint32_t)b;
        }
        o[w] = v;
    }
}

__device__ __forceinline__ double word_pair(const uint32_t* p) { return __hiloint2double((int)p[1], (int)p[0]); }

// checkpoint records -> SoA rows (f64 -> f32 RN, as hgs_scene_upload);
// validates the SH degree words and the quaternions, flips quaternions to
// the canonical hemisphere (data_io.cpp:500-511; negation = sign-bit flip)
__global__ void __launch_bounds__(256) decode_records_kernel(const uint32_t* __restrict__ in, int64_t n, int rows,
                                                             int pre, uint32_t deg, int nq, int q0, int q1,
                                                             float* __restrict__ dst, int64_t cap,
                                                             uint32_t* __restrict__ flags) {
    extern __shared__ uint32_t raw[];  // [cnt][wpr] (wpr odd: conflict-free column reads)
    const int64_t base = (int64_t)blockIdx.x * kTileG;
    const int cnt = (int)(n - base < kTileG ? n - base : (int64_t)kTileG);
    const int wpr = 2 * rows + 1;
    const uint32_t* ip = in + base * wpr;
    for (int w = threadIdx.x; w < cnt * wpr; w += blockDim.x) raw[w] = ip[w];
    __syncthreads();
    uint32_t bad = 0;
    for (int g = threadIdx.x; g < cnt; g += blockDim.x)
        if (raw[g * wpr + 2 * pre] != deg) bad |= CKPT_BAD_DEG;
    for (int i = threadIdx.x; i < nq * kTileG; i += blockDim.x) {
        const int j = i >> 5, g = i & 31;
        if (g >= cnt) continue;
        uint32_t* q = raw + g * wpr + 2 * (j ? q1 : q0);
        const double w = word_pair(q), x = word_pair(q + 2), y = word_pair(q + 4), z = word_pair(q + 6);
        const double s = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(w, w), __dmul_rn(x, x)), __dmul_rn(y, y)),
                                   __dmul_rn(z, z));
        if (!(fabs(__dsqrt_rn(s) - 1.0) <= 1e-6)) bad |= CKPT_NONUNIT;
        const bool flip = w < 0.0 || (w == 0.0 && (x < 0.0 || (x == 0.0 && (y < 0.0 || (y == 0.0 && z < 0.0)))));
        if (flip)
            for (int c = 0; c < 4; ++c) q[2 * c + 1] ^= 0x80000000u;
    }
    if (bad) atomicOr(flags, bad);
    __syncthreads();
    for (int i = threadIdx.x; i < rows * kTileG; i += blockDim.x) {
        const int k = i >> 5, g = i & 31;
        if (g >= cnt) continue;
        const int q = 2 * k + (k >= pre ? 1 : 0);
        dst[(int64_t)k * cap + base + g] = (float)word_pair(raw + g * wpr + q);
    }
}

// rows [r0, r0+dim) of n Gaussians -> f64 Gaussian-major array (AdamBuf m / v)
__global__ void __launch_bounds__(256) encode_rows_kernel(const float* __restrict__ src, int64_t cap, int64_t n, int r0,
                                                          int dim, double* __restrict__ out) {
    extern __shared__ float tile[];  // [dim][kPad]
    const int64_t base = (int64_t)blockIdx.x * kTileG;
    const int cnt = (int)(n - base < kTileG ? n - base : (int64_t)kTileG);
    for (int i = threadIdx.x; i < dim * kTileG; i += blockDim.x) {
        const int k = i >> 5, g = i & 31;
        tile[k * kPad + g] = g < cnt ? src[(int64_t)(r0 + k) * cap + base + g] : 0.f;
    }
    __syncthreads();
    double* o = out + base * dim;
    for (int i = threadIdx.x; i < cnt * dim; i += blockDim.x) {
        const int g = i / dim, k = i - g * dim;
        o[i] = (double)tile[k * kPad + g];
    }
}

__global__ void __launch_bounds__(256) decode_rows_kernel(const double* __restrict__ in, int64_t n, int dim,
                                                          float* __restrict__ dst, int64_t cap, int r0) {
    extern __shared__ float tile[];  // [dim][kPad]
    const int64_t base = (int64_t)blockIdx.x * kTileG;
    const int cnt = (int)(n - base < kTileG ? n - base : (int64_t)kTileG);
    const double* ip = in + base * dim;
    for (int i = threadIdx.x; i < cnt * dim; i += blockDim.x) {
        const int g = i / dim, k = i - g * dim;
        tile[k * kPad + g] = (float)ip[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < dim * kTileG; i += blockDim.x) {
        const int k = i >> 5, g = i & 31;
        if (g < cnt) dst[(int64_t)(r0 + k) * cap + base + g] = tile[k * kPad + g];
    }
}

// densify statistics: accumulated + pending deltas (as hgs_stats_download)
__global__ void encode_stats_kernel(const float* __restrict__ gn, const float* __restrict__ dgn,
                                    const float* __restrict__ cnt, const float* __restrict__ dcnt, int64_t n,
                                    double* __restrict__ gn_out, uint32_t* __restrict__ cnt_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    gn_out[i] = (double)gn[i] + (double)dgn[i];
    cnt_out[i] = (uint32_t)(cnt[i] + dcnt[i]);
}

__global__ void decode_stats_kernel(const double* __restrict__ gn_in, const uint32_t* __restrict__ cnt_in, int64_t n,
                                    float* __restrict__ gn, float* __restrict__ dgn, float* __restrict__ cnt,
                                    float* __restrict__ dcnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    gn[i] = (float)gn_in[i];
    cnt[i] = (float)cnt_in[i];
    dgn[i] = 0.f;
    dcnt[i] = 0.f;
}

// CRC-32 (zlib / IEEE 802.3, reflected 0xEDB88320) of every kCrcChunk-byte
// chunk of [data, data+n), slicing-by-8 from shared-memory tables; the host
// folds the chunk CRCs with zlib's crc32_combine_op.  data is 8-byte aligned.
constexpr uint32_t kCrcChunk = 16384;

__global__ void __launch_bounds__(256) crc32_chunks_kernel(const uint8_t* __restrict__ data, uint64_t n,
                                                           const uint32_t* __restrict__ tables,
                                                           uint32_t* __restrict__ out, uint64_t nchunks) {
    __shared__ uint32_t T[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) T[i >> 8][i & 255] = tables[i];
    __syncthreads();
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint64_t b0 = c * kCrcChunk, b1 = min(n, b0 + kCrcChunk);
    uint32_t crc = 0xFFFFFFFFu;
    uint64_t p = b0;
    for (; p + 8 <= b1; p += 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(data + p);
        const uint32_t lo = w.x ^ crc, hi = w.y;
        crc = T[7][lo & 255] ^ T[6][(lo >> 8) & 255] ^ T[5][(lo >> 16) & 255] ^ T[4][lo >> 24] ^ T[3][hi & 255] ^
              T[2][(hi >> 8) & 255] ^ T[1][(hi >> 16) & 255] ^ T[0][hi >> 24];
    }
    for (; p < b1; ++p) crc = T[0][(crc ^ data[p]) & 255] ^ (crc >> 8);
    out[c] = crc ^ 0xFFFFFFFFu;
}

// header scalars of a payload (4- or 8-byte values at 4-aligned offsets)
struct Patch {
    uint64_t off, val;
    uint32_t bytes, pad;
};
__global__ void patch_kernel(uint8_t* __restrict__ base, const Patch* __restrict__ p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t* w = reinterpret_cast<uint32_t*>(base + p[i].off);
    w[0] = (uint32_t)p[i].val;
    if (p[i].bytes == 8) w[1] = (uint32_t)(p[i].val >> 32);
}

// ------------------------------------------------------------ host layout

struct PoolDesc {
    int rows, pre;
};
PoolDesc pool3(int deg) { return {rows3(deg), R3_SH}; }
PoolDesc pool4(int deg) { return {rows4(deg), R4_SH}; }
uint64_t rec_bytes(const PoolDesc& p) { return 4ull * (2 * p.rows + 1); }

// OPTS classes in file order (data_io.cpp:597-619): pool, first SoA row, dim (-1 = 3K)
struct OptClass {
    bool dyn;
    int r0, dim;
};
const OptClass kOptClasses[12] = {
    {false, R3_MEAN, 3}, {false, R3_Q, 4}, {false, R3_LS, 3}, {false, R3_OP, 1}, {false, R3_SH, -1},
    {true, R4_MEAN, 3},  {true, R4_MT, 1}, {true, R4_QL, 4},  {true, R4_QR, 4},  {true, R4_LS, 4},
    {true, R4_OP, 1},    {true, R4_SH, -1},
};

// byte offsets (within the OPTS payload) of every array's data
struct OptsLayout {
    uint64_t len = 0;
    uint64_t m[12], v[12], n[12];  // data offsets, element counts
    uint64_t gn3, gn4, c3, c4;     // data offsets
    uint64_t n3, n4;
};

OptsLayout opts_layout(uint64_t n3, uint64_t n4, int K3) {
    OptsLayout L;
    uint64_t off = 16;  // step, skipped
    for (int c = 0; c < 12; ++c) {
        const uint64_t cnt = (kOptClasses[c].dyn ? n4 : n3) * (uint64_t)(kOptClasses[c].dim < 0 ? K3 : kOptClasses[c].dim);
        L.n[c] = cnt;
        L.m[c] = off + 8;
        off += 8 + 8 * cnt;
        L.v[c] = off + 8;
        off += 8 + 8 * cnt;
    }
    L.gn3 = off + 8;
    off += 8 + 8 * n3;
    L.gn4 = off + 8;
    off += 8 + 8 * n4;
    L.c3 = off + 8;
    off += 8 + 4 * n3;
    L.c4 = off + 8;
    off += 8 + 4 * n4;
    L.len = off;
    L.n3 = n3;
    L.n4 = n4;
    return L;
}

template <typename T>
void put(uint8_t* p, T v) {
    std::memcpy(p, &v, sizeof(T));
}
template <typename T>
T get(const uint8_t* p) {
    T v;
    std::memcpy(&v, p, sizeof(T));
    return v;
}

void put_scen_header(uint8_t* p, uint32_t deg, double tau, double dur, double ext, uint64_t n3, uint64_t n4) {
    put<uint32_t>(p, deg);
    put<double>(p + 4, tau);
    put<double>(p + 12, dur);
    put<double>(p + 20, ext);
    put<uint64_t>(p + 28, n3);
    put<uint64_t>(p + 36, n4);
}

// the OPTS scalars: step, skipped and every array length
void put_opts_header(uint8_t* p, const OptsLayout& L, uint64_t step, uint64_t skipped) {
    put<uint64_t>(p, step);
    put<uint64_t>(p + 8, skipped);
    for (int c = 0; c < 12; ++c) {
        put<uint64_t>(p + L.m[c] - 8, L.n[c]);
        put<uint64_t>(p + L.v[c] - 8, L.n[c]);
    }
    put<uint64_t>(p + L.gn3 - 8, L.n3);
    put<uint64_t>(p + L.gn4 - 8, L.n4);
    put<uint64_t>(p + L.c3 - 8, L.n3);
    put<uint64_t>(p + L.c4 - 8, L.n4);
}

uint32_t crc_of(const uint8_t* p, uint64_t n) {
    uLong c = crc32_z(0L, Z_NULL, 0);
    return (uint32_t)crc32_z(c, p, (z_size_t)n);
}

void put_section_header(uint8_t* p, const char tag[4], uint64_t len, uint32_t crc) {
    std::memcpy(p, tag, 4);
    put<uint64_t>(p + 4, len);
    put<uint32_t>(p + 12, crc);
}

bool write_file(const char* path, const uint8_t* p, size_t n, IoError& e) {
    FILE* f = std::fopen(path, "wb");
    if (!f) {
        e = {HGS_ERR_FORMAT, std::string("save_checkpoint: cannot open ") + path};
        return false;
    }
    const size_t w = n ? std::fwrite(p, 1, n, f) : 0;
    const bool ok = std::fclose(f) == 0 && w == n;
    if (!ok) e = {HGS_ERR_FORMAT, std::string("save_checkpoint: write failed for ") + path};
    return ok;
}

struct CrcTables {
    uint32_t t[8][256];
    CrcTables() {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
            t[0][i] = c;
        }
        for (int j = 1; j < 8; ++j)
            for (int i = 0; i < 256; ++i) t[j][i] = (t[j - 1][i] >> 8) ^ t[0][t[j - 1][i] & 255];
    }
};

const uint32_t* crc_tables_host() {
    static const CrcTables T;  // thread-safe initialisation
    return &T.t[0][0];
}

uint64_t crc_chunks(uint64_t n) { return (n + kCrcChunk - 1) / kCrcChunk; }

uint32_t crc_combine_chunks(const uint32_t* c, uint64_t n) {
    const uint64_t nch = crc_chunks(n);
    if (nch == 0) return 0u;  // crc32 of the empty string
    const uLong op = crc32_combine_gen((z_off_t)kCrcChunk);
    uLong crc = c[0];
    for (uint64_t i = 1; i < nch; ++i) {
        const uint64_t len = std::min<uint64_t>(kCrcChunk, n - i * kCrcChunk);
        crc = len == kCrcChunk ? crc32_combine_op(crc, c[i], op) : crc32_combine(crc, c[i], (z_off_t)len);
    }
    return (uint32_t)crc;
}

void scen_patches(std::vector<Patch>& v, uint32_t deg, double tau, double dur, double ext, uint64_t n3, uint64_t n4) {
    auto bits = [](double x) {
        uint64_t b;
        std::memcpy(&b, &x, 8);
        return b;
    };
    v.push_back({0, deg, 4, 0});
    v.push_back({4, bits(tau), 8, 0});
    v.push_back({12, bits(dur), 8, 0});
    v.push_back({20, bits(ext), 8, 0});
    v.push_back({28, n3, 8, 0});
    v.push_back({36, n4, 8, 0});
}

void opts_patches(std::vector<Patch>& v, uint64_t base, const OptsLayout& L, uint64_t step, uint64_t skipped) {
    v.push_back({base, step, 8, 0});
    v.push_back({base + 8, skipped, 8, 0});
    for (int c = 0; c < 12; ++c) {
        v.push_back({base + L.m[c] - 8, L.n[c], 8, 0});
        v.push_back({base + L.v[c] - 8, L.n[c], 8, 0});
    }
    v.push_back({base + L.gn3 - 8, L.n3, 8, 0});
    v.push_back({base + L.gn4 - 8, L.n4, 8, 0});
    v.push_back({base + L.c3 - 8, L.n3, 8, 0});
    v.push_back({base + L.c4 - 8, L.n4, 8, 0});
}

int io_threads(uint64_t n) {
    if (n < (16ull << 20)) return 1;
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    return std::min(8, hw);
}

// the file through a shared mapping filled by `io_threads` threads (buffered
// write() calls to one file serialise on its inode lock; page faults on a
// mapping do not), else concurrent pwrite ranges
bool pwrite_file(const char* path, const uint8_t* p, uint64_t n, IoError& e) {
    const int fd = ::open(path, O_RDWR | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) {
        e = {HGS_ERR_FORMAT, std::string("save_checkpoint: cannot open ") + path};
        return false;
    }
    const int T = io_threads(n);
    if (T > 1 && ::ftruncate(fd, (off_t)n) == 0) {
        void* m = ::mmap(nullptr, (size_t)n, PROT_WRITE, MAP_SHARED, fd, 0);
        if (m != MAP_FAILED) {
            const uint64_t part = ((n / T) + 4095) & ~4095ull;
            auto copy = [&](int t) {
                const uint64_t a = std::min(n, (uint64_t)t * part), b = std::min(n, a + part);
                std::memcpy(static_cast<uint8_t*>(m) + a, p + a, (size_t)(b - a));
            };
            std::vector<std::thread> th;
            for (int t = 1; t < T; ++t) th.emplace_back(copy, t);
            copy(0);
            for (auto& x : th) x.join();
            const bool good = ::munmap(m, (size_t)n) == 0 && ::close(fd) == 0;
            if (!good) e = {HGS_ERR_FORMAT, std::string("save_checkpoint: write failed for ") + path};
            return good;
        }
    }
    const uint64_t part = ((n / T) + 4095) & ~4095ull;
    std::vector<char> ok((size_t)T, 1);
    auto work = [&](int t) {
        uint64_t a = (uint64_t)t * part, b = std::min(n, a + part);
        while (a < b) {
            const ssize_t w = ::pwrite(fd, p + a, (size_t)std::min<uint64_t>(b - a, 1ull << 30), (off_t)a);
            if (w <= 0) {
                ok[(size_t)t] = 0;
                return;
            }
            a += (uint64_t)w;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    const bool good = ::close(fd) == 0 && std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
    if (!good) e = {HGS_ERR_FORMAT, std::string("save_checkpoint: write failed for ") + path};
    return good;
}

// ---------------------------------------------------------------- parsing

struct Parsed {
    const uint8_t* scen = nullptr;
    uint64_t scen_len = 0;
    const uint8_t* opts = nullptr;
    uint64_t opts_len = 0;
    bool has_scen = false, has_opts = false;
    // scene header
    uint32_t deg = 0;
    double tau = 0, dur = 0, ext = 0;
    uint64_t n3 = 0, n4 = 0;
    // state
    uint64_t step = 0, skipped = 0;
    OptsLayout L;
};

struct Sec {
    const uint8_t* tag;
    const uint8_t* p;
    uint64_t len;
    uint32_t crc;
};

// data_io.cpp:667-704, structure only: magic, version and every complete
// section header + payload in order.  Returns false (e set) at the first
// structural error; `secs` then holds the complete sections before it (the
// reference checks their checksums before it reaches the error).
bool walk_sections(const uint8_t* b, uint64_t n, const std::string& path, std::vector<Sec>& secs, IoError& e) {
    if (n < 4 || std::memcmp(b, "HGSC", 4) != 0) {
        e = {HGS_ERR_FORMAT, "load_checkpoint: bad magic in " + path};
        return false;
    }
    if (n < 8) {
        e = {HGS_ERR_FORMAT, "load_checkpoint: truncated header in " + path};
        return false;
    }
    const uint32_t version = get<uint32_t>(b + 4);
    if (version != kVersion) {
        e = {HGS_ERR_UNSUPPORTED_VERSION, "load_checkpoint: unsupported version " + std::to_string(version)};
        return false;
    }
    uint64_t off = 8;
    while (off < n) {
        if (n - off < 16) {
            e = {HGS_ERR_FORMAT, "load_checkpoint: truncated section header in " + path};
            return false;
        }
        Sec s{b + off, nullptr, get<uint64_t>(b + off + 4), get<uint32_t>(b + off + 12)};
        off += 16;
        if (s.len > n - off) {
            e = {HGS_ERR_FORMAT, "load_checkpoint: truncated section payload in " + path};
            return false;
        }
        s.p = b + off;
        secs.push_back(s);
        off += s.len;
    }
    return true;
}

// the scene / state sections (the last of each tag wins; unknown tags are
// skipped) and their contents
bool parse_sections(const std::vector<Sec>& secs, const std::string& path, Parsed& P, IoError& e) {
    for (const Sec& s : secs) {
        if (std::memcmp(s.tag, "SCEN", 4) == 0) {
            P.scen = s.p, P.scen_len = s.len, P.has_scen = true;
        } else if (std::memcmp(s.tag, "OPTS", 4) == 0) {
            P.opts = s.p, P.opts_len = s.len, P.has_opts = true;
        }
    }
    if (!P.has_scen) {
        e = {HGS_ERR_FORMAT, "load_checkpoint: no scene section in " + path};
        return false;
    }
    // scene header and exact size (data_io.cpp:553-583: fixed-size records
    // at the scene's SH degree; the per-record degree words are checked by
    // the decoder)
    if (P.scen_len < kScenHdr) {
        e = {HGS_ERR_FORMAT, "checkpoint: truncated section payload"};
        return false;
    }
    P.deg = get<uint32_t>(P.scen);
    if (P.deg > (uint32_t)kMaxDeg) {
        e = {HGS_ERR_FORMAT, "checkpoint: bad scene SH degree"};
        return false;
    }
    P.tau = get<double>(P.scen + 4);
    P.dur = get<double>(P.scen + 12);
    P.ext = get<double>(P.scen + 20);
    P.n3 = get<uint64_t>(P.scen + 28);
    P.n4 = get<uint64_t>(P.scen + 36);
    const uint64_t r3 = rec_bytes(pool3((int)P.deg)), r4 = rec_bytes(pool4((int)P.deg));
    const uint64_t body = P.scen_len - kScenHdr;
    if (P.n3 > body / r3 || P.n4 > (body - P.n3 * r3) / r4) {
        e = {HGS_ERR_FORMAT, "checkpoint: truncated section payload"};
        return false;
    }
    if (P.n3 * r3 + P.n4 * r4 != body) {
        e = {HGS_ERR_FORMAT, "checkpoint: trailing bytes in scene section"};
        return false;
    }
    if (!P.has_opts) return true;
    // state (data_io.cpp:621-643, 705-717): walk the arrays, then require
    // every length to match the scene (the device layout needs them all)
    const uint8_t* s = P.opts;
    const uint64_t sn = P.opts_len;
    uint64_t o = 0;
    auto need = [&](uint64_t k) {
        if (k > sn - o) {
            e = {HGS_ERR_FORMAT, "checkpoint: truncated section payload"};
            return false;
        }
        return true;
    };
    auto arr = [&](uint64_t esz, uint64_t& data, uint64_t& count) {
        if (!need(8)) return false;
        count = get<uint64_t>(s + o);
        o += 8;
        if (count > sn / esz + 1) {
            e = {HGS_ERR_FORMAT, "checkpoint: implausible array length"};
            return false;
        }
        if (!need(count * esz)) return false;
        data = o;
        o += count * esz;
        return true;
    };
    if (!need(16)) return false;
    P.step = get<uint64_t>(s);
    P.skipped = get<uint64_t>(s + 8);
    o = 16;
    const int K3 = 3 * sh_count((int)P.deg);
    const OptsLayout want = opts_layout(P.n3, P.n4, K3);
    bool mismatch = false;
    for (int c = 0; c < 12; ++c) {
        uint64_t dm, cm, dv, cv;
        if (!arr(8, dm, cm) || !arr(8, dv, cv)) return false;
        if (cm != cv) {
            e = {HGS_ERR_FORMAT, "checkpoint: moment size mismatch"};
            return false;
        }
        mismatch |= cm != want.n[c];
        P.L.m[c] = dm, P.L.v[c] = dv, P.L.n[c] = cm;
    }
    uint64_t cg3, cg4, cc3, cc4;
    if (!arr(8, P.L.gn3, cg3) || !arr(8, P.L.gn4, cg4) || !arr(4, P.L.c3, cc3) || !arr(4, P.L.c4, cc4)) return false;
    if (o != sn) {
        e = {HGS_ERR_FORMAT, "checkpoint: trailing bytes in state section"};
        return false;
    }
    mismatch |= cg3 != P.n3 || cg4 != P.n4 || cc3 != P.n3 || cc4 != P.n4;
    if (mismatch) {
        e = {HGS_ERR_FORMAT, "load_checkpoint: optimizer state disagrees with scene in " + path};
        return false;
    }
    P.L.n3 = P.n3, P.L.n4 = P.n4, P.L.len = sn;
    return true;
}

// the whole load check with host checksums (zlib), in the reference's order
bool parse_file(const uint8_t* b, uint64_t n, const std::string& path, Parsed& P, IoError& e) {
    std::vector<Sec> secs;
    IoError walk_err;
    const bool walked = walk_sections(b, n, path, secs, walk_err);
    for (const Sec& s : secs)
        if (crc_of(s.p, s.len) != s.crc) {
            e = {HGS_ERR_INTEGRITY, "load_checkpoint: checksum mismatch in " + path};
            return false;
        }
    if (!walked) {
        e = walk_err;
        return false;
    }
    return parse_sections(secs, path, P, e);
}

bool read_whole(const char* path, std::vector<uint8_t>& buf, IoError& e) {
    FILE* f = path ? std::fopen(path, "rb") : nullptr;
    if (!f) {
        e = {HGS_ERR_FORMAT, std::string("load_checkpoint: cannot open ") + (path ? path : "(null)")};
        return false;
    }
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    buf.resize(sz > 0 ? (size_t)sz : 0);
    const size_t got = buf.empty() ? 0 : std::fread(buf.data(), 1, buf.size(), f);
    std::fclose(f);
    if (got != buf.size()) {
        e = {HGS_ERR_FORMAT, std::string("load_checkpoint: read failed for ") + path};
        return false;
    }
    return true;
}

hgs_status io_fail(const IoError& e) {
    g_io_err = e.msg;
    return e.code;
}

hgs_status ctx_fail(hgs_ctx* ctx, const IoError& e) {
    ctx->err = e.msg;
    return e.code;
}

// ------------------------------------------------------ host-scene records

// host double rows of one Gaussian in record order
struct HostPool {
    const double* f[7];
    int dim[7];
    int nf;  // fields before the SH
};

void host_fields(const hgs_host_scene* s, bool dyn, int K3, HostPool& P) {
    if (dyn) {
        const double* f[7] = {(const double*)s->mean_x, (const double*)s->mean_t, (const double*)s->ql,
                              (const double*)s->qr,     (const double*)s->log_s4, (const double*)s->op4,
                              (const double*)s->sh4};
        const int d[7] = {3, 1, 4, 4, 4, 1, K3};
        for (int i = 0; i < 7; ++i) P.f[i] = f[i], P.dim[i] = d[i];
        P.nf = 6;
    } else {
        const double* f[5] = {(const double*)s->mean3, (const double*)s->quat3, (const double*)s->log_s3,
                              (const double*)s->op3, (const double*)s->sh3};
        const int d[5] = {3, 4, 3, 1, K3};
        for (int i = 0; i < 5; ++i) P.f[i] = f[i], P.dim[i] = d[i];
        P.nf = 4;
    }
}

}  // namespace

// chunk CRCs of [p, p+n) on the context stream (tables uploaded once)
hgs_status crc_launch(hgs_ctx* ctx, const uint8_t* p, uint64_t n, uint32_t* out) {
    const uint64_t nch = crc_chunks(n);
    if (!nch) return HGS_OK;
    if (!ctx->crc_tab.p) {
        CKC(ctx->crc_tab.ensure(8 * 256 * 4));
        CKC(cudaMemcpy(ctx->crc_tab.p, crc_tables_host(), 8 * 256 * 4, cudaMemcpyHostToDevice));
    }
    crc32_chunks_kernel<<<(unsigned)((nch + 255) / 256), 256, 0, ctx->stream>>>(p, n, ctx->crc_tab.as<uint32_t>(), out,
                                                                              nch);
    count_launch();
    CKL();
    return HGS_OK;
}

extern "C" {

const char* hgs_io_last_error(void) { return g_io_err.c_str(); }

// ------------------------------------------------------------ device save
hgs_status hgs_checkpoint_save(hgs_ctx* ctx, const char* path, int with_state) {
    if (!ctx || !path) return HGS_ERR_INVALID_ARGUMENT;
    if (with_state && ctx->state_sharded) {
        ctx->err = "save_checkpoint: the Adam moments are sharded (hgs_gather_state on every rank first)";
        return HGS_ERR_STATE;
    }
    CKC(cudaSetDevice(ctx->device));
    if (!ctx->pipeline.empty()) {
        ctx->err = "save_checkpoint: collect the pipelined iterations first";
        return HGS_ERR_STATE;
    }
    cudaStream_t st = ctx->stream;
    const int deg = ctx->deg, K3 = 3 * sh_count(deg);
    const uint64_t n3 = (uint64_t)ctx->n3, n4 = (uint64_t)ctx->n4;
    const PoolDesc P3 = pool3(deg), P4 = pool4(deg);
    const uint64_t scen_len = kScenHdr + n3 * rec_bytes(P3) + n4 * rec_bytes(P4);
    const OptsLayout L = opts_layout(n3, n4, K3);
    const uint64_t opts_len = with_state ? L.len : 0;
    const uint64_t dev_opts = (scen_len + 255) & ~255ull;
    const uint64_t file_len = 8 + 16 + scen_len + (with_state ? 16 + opts_len : 0);
    uint64_t skipped = 0;
    if (with_state) {
        hgs_status r = hgs_skipped_total(ctx, &skipped, nullptr);
        if (r != HGS_OK) return r;
    }
    const uint64_t nch_s = crc_chunks(scen_len), nch_o = crc_chunks(opts_len);
    const uint64_t dev_crc = (dev_opts + opts_len + 255) & ~255ull;
    const uint64_t dev_patch = (dev_crc + 4 * (nch_s + nch_o) + 255) & ~255ull;
    constexpr int kMaxPatches = 64;
    CKC(ctx->ckpt.ensure(dev_patch + kMaxPatches * sizeof(Patch)));
    uint8_t* d = ctx->ckpt.as<uint8_t>();
    const int nthr = 256;
    auto launch_records = [&](const float* src, int64_t cap, uint64_t n, const PoolDesc& p, uint64_t off) {
        if (!n) return cudaSuccess;
        encode_records_kernel<<<(unsigned)((n + kTileG - 1) / kTileG), nthr, (size_t)p.rows * kPad * 4, st>>>(
            src, cap, (int64_t)n, p.rows, p.pre, (uint32_t)deg, reinterpret_cast<uint32_t*>(d + off));
        count_launch();
        return cudaGetLastError();
    };
    CKC(launch_records(ctx->p3.as<float>(), ctx->cap3, n3, P3, kScenHdr));
    CKC(launch_records(ctx->p4.as<float>(), ctx->cap4, n4, P4, kScenHdr + n3 * rec_bytes(P3)));
    if (with_state) {
        uint8_t* o = d + dev_opts;
        for (int c = 0; c < 12; ++c) {
            const OptClass& k = kOptClasses[c];
            const uint64_t n = k.dyn ? n4 : n3;
            if (!n) continue;
            const int dim = k.dim < 0 ? K3 : k.dim;
            const int64_t cap = k.dyn ? ctx->cap4 : ctx->cap3;
            const float* m = (k.dyn ? ctx->m4 : ctx->m3).as<float>();
            const float* v = (k.dyn ? ctx->v4 : ctx->v3).as<float>();
            const unsigned blocks = (unsigned)((n + kTileG - 1) / kTileG);
            const size_t smem = (size_t)dim * kPad * 4;
            encode_rows_kernel<<<blocks, nthr, smem, st>>>(m, cap, (int64_t)n, k.r0, dim,
                                                           reinterpret_cast<double*>(o + L.m[c]));
            encode_rows_kernel<<<blocks, nthr, smem, st>>>(v, cap, (int64_t)n, k.r0, dim,
                                                           reinterpret_cast<double*>(o + L.v[c]));
            count_launch(2);
            CKL();
        }
        if (n3) {
            encode_stats_kernel<<<(unsigned)((n3 + 255) / 256), 256, 0, st>>>(
                ctx->gn3.as<float>(), ctx->dgn3, ctx->cnt3.as<float>(), ctx->dcnt3, (int64_t)n3,
                reinterpret_cast<double*>(o + L.gn3), reinterpret_cast<uint32_t*>(o + L.c3));
            count_launch();
        }
        if (n4) {
            encode_stats_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(
                ctx->gn4.as<float>(), ctx->dgn4, ctx->cnt4.as<float>(), ctx->dcnt4, (int64_t)n4,
                reinterpret_cast<double*>(o + L.gn4), reinterpret_cast<uint32_t*>(o + L.c4));
            count_launch();
        }
        CKL();
    }
    // header scalars written into the device payloads, then the CRC-32 of
    // both sections on the device (chunk CRCs, folded on the host)
    const uint64_t h_crc = (file_len + 255) & ~255ull;
    const uint64_t h_patch = (h_crc + 4 * (nch_s + nch_o) + 255) & ~255ull;
    CKC(ctx->ckpt_host.ensure(h_patch + kMaxPatches * sizeof(Patch)));
    uint8_t* h = static_cast<uint8_t*>(ctx->ckpt_host.p);
    std::vector<Patch> patches;
    scen_patches(patches, (uint32_t)deg, ctx->tau, ctx->duration, ctx->extent, n3, n4);
    if (with_state) opts_patches(patches, dev_opts, L, ctx->step, skipped);
    std::memcpy(h + h_patch, patches.data(), patches.size() * sizeof(Patch));
    CKC(cudaMemcpyAsync(d + dev_patch, h + h_patch, patches.size() * sizeof(Patch), cudaMemcpyHostToDevice, st));
    patch_kernel<<<1, kMaxPatches, 0, st>>>(d, reinterpret_cast<const Patch*>(d + dev_patch), (int)patches.size());
    count_launch();
    hgs_status r = crc_launch(ctx, d, scen_len, reinterpret_cast<uint32_t*>(d + dev_crc));
    if (r != HGS_OK) return r;
    if (with_state) {
        r = crc_launch(ctx, d + dev_opts, opts_len, reinterpret_cast<uint32_t*>(d + dev_crc) + nch_s);
        if (r != HGS_OK) return r;
    }
    uint8_t* hs = h + 24;
    uint8_t* ho = hs + scen_len + 16;
    CKC(cudaMemcpyAsync(hs, d, scen_len, cudaMemcpyDeviceToHost, st));
    if (with_state && opts_len) CKC(cudaMemcpyAsync(ho, d + dev_opts, opts_len, cudaMemcpyDeviceToHost, st));
    CKC(cudaMemcpyAsync(h + h_crc, d + dev_crc, 4 * (nch_s + nch_o), cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    const uint32_t* hc = reinterpret_cast<const uint32_t*>(h + h_crc);
    std::memcpy(h, "HGSC", 4);
    put<uint32_t>(h + 4, kVersion);
    put_section_header(h + 8, "SCEN", scen_len, crc_combine_chunks(hc, scen_len));
    if (with_state) put_section_header(ho - 16, "OPTS", opts_len, crc_combine_chunks(hc + nch_s, opts_len));
    IoError e;
    if (!pwrite_file(path, h, file_len, e)) return ctx_fail(ctx, e);
    return HGS_OK;
}

// ------------------------------------------------------------ device load
hgs_status hgs_checkpoint_load(hgs_ctx* ctx, const char* path, int* has_state) {
    if (!ctx || !path) return HGS_ERR_INVALID_ARGUMENT;
    ctx->state_sharded = false;  // the loaded state is whole
    CKC(cudaSetDevice(ctx->device));
    IoError e;
    // the file into pinned memory (concurrent pread ranges)
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return ctx_fail(ctx, {HGS_ERR_FORMAT, std::string("load_checkpoint: cannot open ") + path});
    struct stat sb;
    const uint64_t n = ::fstat(fd, &sb) == 0 && sb.st_size > 0 ? (uint64_t)sb.st_size : 0;
    const uint64_t nch_max = 2 * crc_chunks(n) + 2;
    const uint64_t h_crc = (n + 255) & ~255ull;
    if (cudaError_t ce = ctx->ckpt_host.ensure(h_crc + 4 * nch_max); ce != cudaSuccess) {
        ::close(fd);
        CKC(ce);
    }
    uint8_t* h = static_cast<uint8_t*>(ctx->ckpt_host.p);
    {
        const int T = io_threads(n);
        const uint64_t part = ((n / T) + 4095) & ~4095ull;
        std::vector<char> ok((size_t)T, 1);
        auto work = [&](int t) {
            uint64_t a = (uint64_t)t * part, b = std::min(n, a + part);
            while (a < b) {
                const ssize_t got = ::pread(fd, h + a, (size_t)std::min<uint64_t>(b - a, 1ull << 30), (off_t)a);
                if (got <= 0) {
                    ok[(size_t)t] = 0;
                    return;
                }
                a += (uint64_t)got;
            }
        };
        std::vector<std::thread> th;
        for (int t = 1; t < T; ++t) th.emplace_back(work, t);
        work(0);
        for (auto& x : th) x.join();
        ::close(fd);
        if (!std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; }))
            return ctx_fail(ctx, {HGS_ERR_FORMAT, std::string("load_checkpoint: read failed for ") + path});
    }
    std::vector<Sec> secs;
    IoError walk_err;
    const bool walked = walk_sections(h, n, path, secs, walk_err);
    // the sections the device decodes (the last of each tag) are checksummed
    // on the device after their upload, every other one on the host
    int is = -1, io = -1;
    for (int i = 0; i < (int)secs.size(); ++i) {
        if (std::memcmp(secs[i].tag, "SCEN", 4) == 0) is = i;
        if (std::memcmp(secs[i].tag, "OPTS", 4) == 0) io = i;
    }
    cudaStream_t st = ctx->stream;
    const uint64_t scen_len = is >= 0 ? secs[is].len : 0, opts_len = io >= 0 ? secs[io].len : 0;
    const uint64_t dev_opts = (scen_len + 255) & ~255ull;
    const uint64_t nch_s = crc_chunks(scen_len), nch_o = crc_chunks(opts_len);
    const uint64_t dev_crc = (dev_opts + opts_len + 255) & ~255ull;
    CKC(ctx->ckpt.ensure(dev_crc + 4 * (nch_s + nch_o) + 256));
    uint8_t* d = ctx->ckpt.as<uint8_t>();
    if (scen_len) CKC(cudaMemcpyAsync(d, secs[is].p, scen_len, cudaMemcpyHostToDevice, st));
    if (opts_len) CKC(cudaMemcpyAsync(d + dev_opts, secs[io].p, opts_len, cudaMemcpyHostToDevice, st));
    hgs_status r = crc_launch(ctx, d, scen_len, reinterpret_cast<uint32_t*>(d + dev_crc));
    if (r != HGS_OK) return r;
    r = crc_launch(ctx, d + dev_opts, opts_len, reinterpret_cast<uint32_t*>(d + dev_crc) + nch_s);
    if (r != HGS_OK) return r;
    uint32_t* hc = reinterpret_cast<uint32_t*>(h + h_crc);
    if (nch_s + nch_o) CKC(cudaMemcpyAsync(hc, d + dev_crc, 4 * (nch_s + nch_o), cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    for (int i = 0; i < (int)secs.size(); ++i) {  // in file order, like the reference
        const uint32_t crc = i == is   ? crc_combine_chunks(hc, scen_len)
                             : i == io ? crc_combine_chunks(hc + nch_s, opts_len)
                                       : crc_of(secs[i].p, secs[i].len);
        if (crc != secs[i].crc)
            return ctx_fail(ctx, {HGS_ERR_INTEGRITY, std::string("load_checkpoint: checksum mismatch in ") + path});
    }
    if (!walked) return ctx_fail(ctx, walk_err);
    Parsed P;
    if (!parse_sections(secs, path, P, e)) return ctx_fail(ctx, e);
    // replace the device scene (zeroed optimizer state and statistics)
    r = hgs_scene_alloc(ctx, (int64_t)P.n4, (int64_t)P.n3, (int)P.deg, P.tau, P.ext, P.dur);
    if (r != HGS_OK) return r;
    CKC(ctx->counters.ensure(sizeof(Counters)));
    uint32_t* dflags = &ctx->counters.as<Counters>()->flags;
    CKC(cudaMemsetAsync(dflags, 0, 4, st));
    const int deg = (int)P.deg, K3 = 3 * sh_count(deg);
    const PoolDesc P3 = pool3(deg), P4 = pool4(deg);
    auto launch_records = [&](float* dst, int64_t cap, uint64_t cnt, const PoolDesc& p, uint64_t off, int nq, int q0,
                              int q1) {
        if (!cnt) return cudaSuccess;
        decode_records_kernel<<<(unsigned)((cnt + kTileG - 1) / kTileG), 256, (size_t)kTileG * (2 * p.rows + 1) * 4, st>>>(
            reinterpret_cast<const uint32_t*>(d + off), (int64_t)cnt, p.rows, p.pre, (uint32_t)deg, nq, q0, q1, dst,
            cap, dflags);
        count_launch();
        return cudaGetLastError();
    };
    CKC(launch_records(ctx->p3.as<float>(), ctx->cap3, P.n3, P3, kScenHdr, 1, R3_Q, R3_Q));
    CKC(launch_records(ctx->p4.as<float>(), ctx->cap4, P.n4, P4, kScenHdr + P.n3 * rec_bytes(P3), 2, R4_QL, R4_QR));
    if (P.has_opts) {
        const uint8_t* o = d + dev_opts;
        for (int c = 0; c < 12; ++c) {
            const OptClass& k = kOptClasses[c];
            const uint64_t cnt = k.dyn ? P.n4 : P.n3;
            if (!cnt) continue;
            const int dim = k.dim < 0 ? K3 : k.dim;
            const int64_t cap = k.dyn ? ctx->cap4 : ctx->cap3;
            float* m = (k.dyn ? ctx->m4 : ctx->m3).as<float>();
            float* v = (k.dyn ? ctx->v4 : ctx->v3).as<float>();
            const unsigned blocks = (unsigned)((cnt + kTileG - 1) / kTileG);
            const size_t smem = (size_t)dim * kPad * 4;
            decode_rows_kernel<<<blocks, 256, smem, st>>>(reinterpret_cast<const double*>(o + P.L.m[c]), (int64_t)cnt,
                                                          dim, m, cap, k.r0);
            decode_rows_kernel<<<blocks, 256, smem, st>>>(reinterpret_cast<const double*>(o + P.L.v[c]), (int64_t)cnt,
                                                          dim, v, cap, k.r0);
            count_launch(2);
            CKL();
        }
        if (P.n3) {
            decode_stats_kernel<<<(unsigned)((P.n3 + 255) / 256), 256, 0, st>>>(
                reinterpret_cast<const double*>(o + P.L.gn3), reinterpret_cast<const uint32_t*>(o + P.L.c3),
                (int64_t)P.n3, ctx->gn3.as<float>(), ctx->dgn3, ctx->cnt3.as<float>(), ctx->dcnt3);
            count_launch();
        }
        if (P.n4) {
            decode_stats_kernel<<<(unsigned)((P.n4 + 255) / 256), 256, 0, st>>>(
                reinterpret_cast<const double*>(o + P.L.gn4), reinterpret_cast<const uint32_t*>(o + P.L.c4),
                (int64_t)P.n4, ctx->gn4.as<float>(), ctx->dgn4, ctx->cnt4.as<float>(), ctx->dcnt4);
            count_launch();
        }
        CKL();
    }
    uint32_t* hf = reinterpret_cast<uint32_t*>(h);  // the file image is no longer needed
    CKC(cudaMemcpyAsync(hf, dflags, 4, cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    const uint32_t flags = *hf;
    if (flags) {
        // leave an empty, consistent scene behind rather than a half-decoded one
        hgs_scene_alloc(ctx, 0, 0, deg, P.tau, P.ext, P.dur);
        if (flags & CKPT_BAD_DEG)
            return ctx_fail(ctx, {HGS_ERR_FORMAT, "checkpoint: SH degree of a Gaussian differs from the scene's"});
        return ctx_fail(ctx, {HGS_ERR_FORMAT, "checkpoint: non-unit quaternion"});
    }
    if (P.has_opts) {
        ctx->step = P.step;
        r = hgs_skipped_total(ctx, nullptr, &P.skipped);
        if (r != HGS_OK) return r;
    }
    if (has_state) *has_state = P.has_opts ? 1 : 0;
    return HGS_OK;
}

// ------------------------------------------------------------- host scenes
hgs_status hgs_checkpoint_write(const hgs_host_scene* s, const hgs_host_state* st, const char* path) {
    if (!s || !path || s->n3 < 0 || s->n4 < 0 || s->sh_degree < 0 || s->sh_degree > kMaxDeg) {
        g_io_err = "save_checkpoint: bad arguments";
        return HGS_ERR_INVALID_ARGUMENT;
    }
    const int deg = s->sh_degree, K3 = 3 * sh_count(deg);
    const uint64_t n3 = (uint64_t)s->n3, n4 = (uint64_t)s->n4;
    const uint64_t r3 = rec_bytes(pool3(deg)), r4 = rec_bytes(pool4(deg));
    const uint64_t scen_len = kScenHdr + n3 * r3 + n4 * r4;
    const OptsLayout L = opts_layout(n3, n4, K3);
    const uint64_t file_len = 24 + scen_len + (st ? 16 + L.len : 0);
    std::vector<uint8_t> buf(file_len);
    uint8_t* h = buf.data();
    uint8_t* hs = h + 24;
    std::memcpy(h, "HGSC", 4);
    put<uint32_t>(h + 4, kVersion);
    put_scen_header(hs, (uint32_t)deg, s->tau, s->duration_seconds, s->extent, n3, n4);
    uint8_t* p = hs + kScenHdr;
    for (int pool = 0; pool < 2; ++pool) {  // statics first (data_io.cpp:534-550)
        const bool dyn = pool == 1;
        HostPool hp;
        host_fields(s, dyn, K3, hp);
        const uint64_t n = dyn ? n4 : n3;
        for (int fi = 0; fi <= hp.nf; ++fi)
            if (n && !hp.f[fi]) {
                g_io_err = "save_checkpoint: null field pointer";
                return HGS_ERR_INVALID_ARGUMENT;
            }
        for (uint64_t i = 0; i < n; ++i) {
            for (int fi = 0; fi <= hp.nf; ++fi) {
                if (fi == hp.nf) {
                    put<uint32_t>(p, (uint32_t)deg);
                    p += 4;
                }
                std::memcpy(p, hp.f[fi] + i * hp.dim[fi], 8 * (size_t)hp.dim[fi]);
                p += 8 * (size_t)hp.dim[fi];
            }
        }
    }
    put_section_header(h + 8, "SCEN", scen_len, crc_of(hs, scen_len));
    if (st) {
        uint8_t* o = hs + scen_len + 16;
        put_opts_header(o, L, st->step, st->skipped_nonfinite);
        for (int c = 0; c < 12; ++c) {
            const bool dyn = kOptClasses[c].dyn;
            HostPool pm, pv;
            host_fields(&st->m, dyn, K3, pm);
            host_fields(&st->v, dyn, K3, pv);
            const int fi = dyn ? c - 5 : c;
            if (L.n[c] && (!pm.f[fi] || !pv.f[fi])) {
                g_io_err = "save_checkpoint: null optimizer-state pointer";
                return HGS_ERR_INVALID_ARGUMENT;
            }
            if (L.n[c]) {
                std::memcpy(o + L.m[c], pm.f[fi], 8 * L.n[c]);
                std::memcpy(o + L.v[c], pv.f[fi], 8 * L.n[c]);
            }
        }
        if ((n3 && (!st->grad_norm3 || !st->count3)) || (n4 && (!st->grad_norm4 || !st->count4))) {
            g_io_err = "save_checkpoint: null statistics pointer";
            return HGS_ERR_INVALID_ARGUMENT;
        }
        if (n3) std::memcpy(o + L.gn3, st->grad_norm3, 8 * n3);
        if (n4) std::memcpy(o + L.gn4, st->grad_norm4, 8 * n4);
        if (n3) std::memcpy(o + L.c3, st->count3, 4 * n3);
        if (n4) std::memcpy(o + L.c4, st->count4, 4 * n4);
        put_section_header(o - 16, "OPTS", L.len, crc_of(o, L.len));
    }
    IoError e;
    if (!write_file(path, h, file_len, e)) return io_fail(e);
    return HGS_OK;
}

hgs_status hgs_checkpoint_info(const char* path, int64_t* n4, int64_t* n3, int32_t* deg, int* has_state) {
    std::vector<uint8_t> buf;
    IoError e;
    Parsed P;
    if (!read_whole(path, buf, e) || !parse_file(buf.data(), buf.size(), path, P, e)) return io_fail(e);
    if (n4) *n4 = (int64_t)P.n4;
    if (n3) *n3 = (int64_t)P.n3;
    if (deg) *deg = (int32_t)P.deg;
    if (has_state) *has_state = P.has_opts ? 1 : 0;
    return HGS_OK;
}

hgs_status hgs_checkpoint_read(const char* path, hgs_host_scene* out, hgs_host_state* st) {
    if (!out) {
        g_io_err = "load_checkpoint: null output";
        return HGS_ERR_INVALID_ARGUMENT;
    }
    std::vector<uint8_t> buf;
    IoError e;
    Parsed P;
    if (!read_whole(path, buf, e) || !parse_file(buf.data(), buf.size(), path, P, e)) return io_fail(e);
    if ((uint64_t)out->n3 != P.n3 || (uint64_t)out->n4 != P.n4 || out->sh_degree != (int32_t)P.deg) {
        g_io_err = "load_checkpoint: output buffers sized for a different scene (use hgs_checkpoint_info)";
        return HGS_ERR_INVALID_ARGUMENT;
    }
    const int deg = (int)P.deg, K3 = 3 * sh_count(deg);
    const uint8_t* p = P.scen + kScenHdr;
    for (int pool = 0; pool < 2; ++pool) {
        const bool dyn = pool == 1;
        HostPool hp;
        host_fields(out, dyn, K3, hp);
        const uint64_t n = dyn ? P.n4 : P.n3;
        for (int fi = 0; fi <= hp.nf; ++fi)
            if (n && !hp.f[fi]) {
                g_io_err = "load_checkpoint: null field pointer";
                return HGS_ERR_INVALID_ARGUMENT;
            }
        for (uint64_t i = 0; i < n; ++i) {
            for (int fi = 0; fi <= hp.nf; ++fi) {
                if (fi == hp.nf) {
                    const uint32_t d = get<uint32_t>(p);
                    p += 4;
                    if (d > (uint32_t)kMaxDeg) return io_fail({HGS_ERR_FORMAT, "checkpoint: bad SH degree"});
                    if (d != P.deg)
                        return io_fail(
                            {HGS_ERR_FORMAT, "checkpoint: SH degree of a Gaussian differs from the scene's"});
                }
                double* dst = const_cast<double*>(hp.f[fi]) + i * hp.dim[fi];
                std::memcpy(dst, p, 8 * (size_t)hp.dim[fi]);
                p += 8 * (size_t)hp.dim[fi];
                const bool quat = dyn ? (fi == 2 || fi == 3) : fi == 1;
                if (quat) {  // data_io.cpp:500-511
                    const double w = dst[0], x = dst[1], y = dst[2], z = dst[3];
                    const double nrm = std::sqrt(w * w + x * x + y * y + z * z);
                    if (!(std::fabs(nrm - 1.0) <= 1e-6))
                        return io_fail({HGS_ERR_FORMAT, "checkpoint: non-unit quaternion"});
                    const bool flip =
                        w < 0.0 || (w == 0.0 && (x < 0.0 || (x == 0.0 && (y < 0.0 || (y == 0.0 && z < 0.0)))));
                    if (flip)
                        for (int c = 0; c < 4; ++c) dst[c] = -dst[c];
                }
            }
        }
    }
    out->tau = P.tau;
    out->extent = P.ext;
    out->duration_seconds = P.dur;
    if (st && P.has_opts) {
        const uint8_t* o = P.opts;
        st->step = P.step;
        st->skipped_nonfinite = P.skipped;
        for (int c = 0; c < 12; ++c) {
            const bool dyn = kOptClasses[c].dyn;
            HostPool pm, pv;
            host_fields(&st->m, dyn, K3, pm);
            host_fields(&st->v, dyn, K3, pv);
            const int fi = dyn ? c - 5 : c;
            if (!P.L.n[c]) continue;
            if (!pm.f[fi] || !pv.f[fi]) {
                g_io_err = "load_checkpoint: null optimizer-state pointer";
                return HGS_ERR_INVALID_ARGUMENT;
            }
            std::memcpy(const_cast<double*>(pm.f[fi]), o + P.L.m[c], 8 * P.L.n[c]);
            std::memcpy(const_cast<double*>(pv.f[fi]), o + P.L.v[c], 8 * P.L.n[c]);
        }
        if ((P.n3 && (!st->grad_norm3 || !st->count3)) || (P.n4 && (!st->grad_norm4 || !st->count4))) {
            g_io_err = "load_checkpoint: null statistics pointer";
            return HGS_ERR_INVALID_ARGUMENT;
        }
        if (P.n3) std::memcpy(st->grad_norm3, o + P.L.gn3, 8 * P.n3);
        if (P.n4) std::memcpy(st->grad_norm4, o + P.L.gn4, 8 * P.n4);
        if (P.n3) std::memcpy(st->count3, o + P.L.c3, 4 * P.n3);
        if (P.n4) std::memcpy(st->count4, o + P.L.c4, 4 * P.n4);
    }
    return HGS_OK;
}

}  // extern "C"
