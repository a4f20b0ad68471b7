// Microbenchmark: the access-pattern ceiling of a high pass that keeps the
// signal as int32 in registers (the compact plan's int32 -> int32 pass with
// twice the elements per CTA): 256 threads x 64 int32 per CTA (2^14), lanes
// on 32 consecutive int32 (128-byte segments), warps and registers on rows
// at stride 2^(k+1) int32 slots, read from one half-block layout and written
// to the other (no butterflies, no exchange).  Compared with the same walk
// at 32 registers per thread (2^13 int32 per CTA: the u64 engine's tile).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_int32 tools/mb_int32.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// R register bits per thread (E = 2^R int32), 3 warp bits, 5 lane bits.
// Tile rows: warp bits then register bits; row stride = 2^(k+1) int32.
template <int R>
__global__ void __launch_bounds__(256, 2) k_walk32(const int* __restrict__ src, int* __restrict__ dst, int k, int n) {
    constexpr int E = 1 << R;
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // tile id -> free bits: rows occupy row bits [0, 3 + R) at stride 2^(k+1);
    // the tile id's low bits take the column groups between 32 and 2^(k+1)
    // (k+1-5 bits), the rest goes above the rows.
    const uint64_t tile = blockIdx.x;
    const int mid = k + 1 - 5;
    const uint64_t base = ((tile & ((1ull << mid) - 1)) << 5) | ((tile >> mid) << (k + 1 + 3 + R));
    const uint64_t t0 = base + lane + ((uint64_t)warp << (k + 1));
    int v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = __ldcg(src + t0 + ((uint64_t)j << (k + 1 + 3)));
#pragma unroll
    for (int j = 0; j < E; ++j) dst[t0 + ((uint64_t)j << (k + 1 + 3))] = v[j] + 1;
}

template <int R>
static void run(int* a, int* b, int n, int k) {
    // n: log2 of the int32 count of each half
    const unsigned grid = 1u << (n - 8 - R);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 2; ++w) k_walk32<R><<<grid, 256>>>(a, b, k, n);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_walk32<R><<<grid, 256>>>(r & 1 ? b : a, r & 1 ? a : b, k, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 8.0 * (double)(1ull << n) * reps;  // 4 read + 4 write per point
    printf("R=%d (%2d int32/thread, 2^%d per CTA) k=%2d: %.3f ms per pass of 2^%d points, %.2f TB/s  %s\n", R, 1 << R,
           8 + R, k, ms / reps, n, bytes / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 32;  // 2^32 int32 points = 16 GiB per half
    int *a = nullptr, *b = nullptr;
    if (cudaMalloc(&a, 4ull << n) != cudaSuccess || cudaMalloc(&b, 4ull << n) != cudaSuccess) return 1;
    cudaMemset(a, 0, 4ull << n);
    cudaMemset(b, 0, 4ull << n);
    for (int k : {13, 18, 22}) {
        run<5>(a, b, n, k);
        run<6>(a, b, n, k);
    }
    return 0;
}
