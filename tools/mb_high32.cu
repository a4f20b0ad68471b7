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

// 9 rows with 16-byte loads and 8-byte stores (the mirror image of CfgHighW<5>):
//   round 0 reg {0,1,5,6,7,8} lane {2,3,4,9,10} warp {11,12,13} stages 5..8
//   round 1 reg {0,9..13}     lane {1..5}       warp {6,7,8}    stages 9..13
struct CfgHighW5B {
    static constexpr int NR = 2;
    BW_HD static constexpr int nreg(int) { return 6; }
    BW_HD static constexpr int reg(int rd, int i) { return bw::nib(rd == 0 ? 0x876510ull : 0xDCBA90ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return bw::nib(rd == 0 ? 0xA9432ull : 0x54321ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return bw::nib(rd == 0 ? 0xDCBull : 0x876ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1E0u : 0x3E00u; }
    BW_HD static constexpr uint32_t slot(uint32_t e) { return e; }
};

template <int L, int MINB, class C = CfgHighW<L>>
static void run(int* x, int n, int k, int reps, const char* what = "") {
    auto kern = k32_high<L, MINB, C>;
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
    printf("k32_high<L=%d>%s %d CTAs/SM asked, %d resident: n=%d stages %d..%d: %.3f ms, %.2f TB/s of 8 B/point  %s\n", L,
           what, MINB, occ, n, k, k + 13 - L, total / reps, 8.0 * (double)(1ull << n) / (total / reps / 1e3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 5;
    int* x = nullptr;
    if (cudaMalloc(&x, 8ull << 32) != cudaSuccess) return 1;
    run<5, 2>(x, 32, 23, reps);
    run<5, 2>(x, 32, 18, reps);
    run<5, 2>(x, 32, 14, reps);
    run<5, 2, CfgHighW5B>(x, 32, 23, reps, " (16-byte loads, 8-byte stores)");
    run<5, 3>(x, 32, 23, reps);
    run<6, 2>(x, 31, 23, reps);
    run<6, 3>(x, 31, 23, reps);
    run<6, 2>(x, 32, 24, reps);
    run<6, 3>(x, 32, 24, reps);
    return 0;
}
