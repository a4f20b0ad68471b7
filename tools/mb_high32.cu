// Microbenchmark: the compact plan's int32 -> int32 high pass (k32_high,
// bw_kernels32.cuh) with two and three CTAs per SM, 9 rows (L = 5, n = 32:
// stages 23..31) and 8 rows (L = 6, n = 31: stages 23..30), 8 bytes per point.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_1607_01039_b200/csrc -Iinclude \
//        -o tools/bin/mb_high32 tools/mb_high32.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "bw_kernels32.cuh"

using namespace bw::w32;

__global__ void k_fill32(int* x, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        x[i] = (int)(h % 1025) - 512;
    }
}

template <int L, int MINB>
static void run(int* x, int n, int k, int reps) {
    auto kern = k32_high<L, MINB>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kNT, kSmemBytes);
    const unsigned grid = 1u << (n - kBits);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float total = 0;
    for (int r = 0; r < reps + 1; ++r) {
        k_fill32<<<148 * 8, 256>>>(x, 2ull << n);
        cudaEventRecord(e0);
        kern<<<grid, kNT, kSmemBytes>>>(reinterpret_cast<const uint32_t*>(x) + (1u << 14), reinterpret_cast<uint32_t*>(x), k);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r) total += ms;
    }
    printf("k32_high<L=%d> %d CTAs/SM asked, %d resident: n=%d stages %d..%d: %.3f ms, %.2f TB/s of 8 B/point  %s\n", L, MINB,
           occ, n, k, k + 13 - L, total / reps, 8.0 * (double)(1ull << n) / (total / reps / 1e3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 5;
    int* x = nullptr;
    if (cudaMalloc(&x, 8ull << 32) != cudaSuccess) return 1;
    run<5, 2>(x, 32, 23, reps);
    run<5, 3>(x, 32, 23, reps);
    run<6, 2>(x, 31, 23, reps);
    run<6, 3>(x, 31, 23, reps);
    run<6, 2>(x, 32, 24, reps);
    run<6, 3>(x, 32, 24, reps);
    return 0;
}
