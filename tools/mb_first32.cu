// Microbenchmark: load-phase variants of the compact plan's first pass
// (k32_first, bw_kernels32.cuh) on a +-1 signal of 2^n int64 (n = 32: the
// config-4 pass, 12 bytes per point): plain and checked, VAR 0 / 1 / 2 / 3.
// Each launch starts from the regenerated input; a checksum of the int32
// half every variant writes must agree.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1607_01039_b200/csrc -Iinclude \
//        -o tools/bin/mb_first32 tools/mb_first32.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "bw_kernels32.cuh"

using namespace bw::w32;

__global__ void k_fill(long long* x, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        x[i] = 1 - 2 * (long long)(h & 1);
    }
}

// sum over the int32 half the pass wrote (half h of every 2^15-slot block)
__global__ void k_sum_half(const uint32_t* x, uint64_t nslots, int half, unsigned long long* out) {
    unsigned long long s = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nslots; i += (uint64_t)gridDim.x * blockDim.x)
        if (((i >> 14) & 1) == (uint64_t)half) s += (unsigned long long)x[i] * (2 * (i & 0xffff) + 1);
    atomicAdd(out, s);
}

template <int L, int MODE, int VAR>
static void run(long long* x, int n, unsigned* flags, unsigned* abort, unsigned long long* sum, int reps) {
    auto kern = k32_first<L, MODE, VAR>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    const unsigned grid = 1u << (n - kBits);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float total = 0, best = 1e9f;
    for (int r = 0; r < reps + 1; ++r) {
        k_fill<<<148 * 8, 256>>>(x, 1ull << n);
        cudaMemset(flags, 0, 4ull << (n - kBits));
        cudaMemset(abort, 0, 4);
        cudaEventRecord(e0);
        kern<<<grid, kNT, kSmemBytes>>>(reinterpret_cast<const unsigned long long*>(x), reinterpret_cast<uint32_t*>(x), 14,
                                        7u, flags, abort);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r) {
            total += ms;
            best = ms < best ? ms : best;
        }
    }
    cudaMemset(sum, 0, 8);
    k_sum_half<<<148 * 8, 256>>>(reinterpret_cast<const uint32_t*>(x), 2ull << n, 0, sum);
    unsigned long long h = 0;
    unsigned ab = 0;
    cudaMemcpy(&h, sum, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ab, abort, 4, cudaMemcpyDeviceToHost);
    const double bytes = 12.0 * (double)(1ull << n);
    printf("L=%d %s VAR=%d: mean %.3f ms, best %.3f ms, %.2f TB/s of 12 B/point  abort=%u checksum=%016llx  %s\n", L,
           MODE ? "checked" : "plain  ", VAR, total / reps, best, bytes / (total / reps / 1e3) / 1e12, ab, h,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 32;
    const int reps = argc > 2 ? atoi(argv[2]) : 5;
    long long* x = nullptr;
    unsigned *flags = nullptr, *abort = nullptr;
    unsigned long long* sum = nullptr;
    if (cudaMalloc(&x, 8ull << n) != cudaSuccess) return 1;
    cudaMalloc(&flags, 4ull << (n - kBits));
    cudaMalloc(&abort, 4);
    cudaMalloc(&sum, 8);
    run<5, 0, 0>(x, n, flags, abort, sum, reps);
    run<5, 0, 2>(x, n, flags, abort, sum, reps);
    run<5, 1, 0>(x, n, flags, abort, sum, reps);
    run<5, 1, 1>(x, n, flags, abort, sum, reps);
    run<5, 1, 2>(x, n, flags, abort, sum, reps);
    run<5, 1, 3>(x, n, flags, abort, sum, reps);
    run<5, 1, 4>(x, n, flags, abort, sum, reps);
    run<6, 0, 0>(x, n - 1, flags, abort, sum, reps);
    run<6, 0, 2>(x, n - 1, flags, abort, sum, reps);
    run<6, 1, 0>(x, n - 1, flags, abort, sum, reps);
    run<6, 1, 2>(x, n - 1, flags, abort, sum, reps);
    run<6, 1, 3>(x, n - 1, flags, abort, sum, reps);
    run<6, 1, 4>(x, n - 1, flags, abort, sum, reps);
    return 0;
}
