// Bit-exactness of gm::Rcp (shared-reciprocal FP64 division, gauss_math.cuh) against IEEE
// division on random operands; tests/test_gpu_div.py builds and runs it on the GPU.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include "../paper_2505_13215_b200/csrc/gauss_math.cuh"
using namespace hgs::gm;
__device__ uint64_t mix(uint64_t x) { x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x; }
__global__ void k(uint64_t seed, unsigned long long* bad, int mode) {
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t h1 = mix(seed * 0x9E3779B97F4A7C15ULL + i), h2 = mix(h1 + 12345);
    double a, b;
    if (mode == 0) {  // random bit patterns (finite)
        a = __longlong_as_double(h1 & 0x7fefffffffffffffULL); b = __longlong_as_double(h2 & 0x7fefffffffffffffULL);
        if (h1 >> 63) a = -a;
    } else {  // moderate magnitudes like the geometry
        a = ((double)(h1 >> 11) / 9007199254740992.0 - 0.5) * exp2((double)((int)(h1 % 60) - 30));
        b = ((double)(h2 >> 11) / 9007199254740992.0 + 1e-3) * exp2((double)((int)(h2 % 60) - 30));
    }
    volatile double bb = b;
    double ref = a / bb;
    Rcp r(b);
    double q = r.div(a);
    if (__double_as_longlong(q) != __double_as_longlong(ref) && !(isnan(q) && isnan(ref))) atomicAdd(bad, 1ull);
}
int main(int argc, char** argv) {
    const int rounds = argc > 1 ? atoi(argv[1]) : 50;
    unsigned long long* d; cudaMalloc(&d, 8); 
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(d, 0, 8);
        for (int s = 0; s < rounds; ++s) k<<<65536, 256>>>(s + 1000 * mode, d, mode);
        unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %llu mismatches of %llu\n", mode, h, (unsigned long long)rounds * 65536 * 256);
    }
    return 0;
}
