// Microbenchmark: HBM efficiency of the high-pass access pattern without any
// compute.  A CTA (256 threads, 32 int64 per thread = 2^13 elements) reads a
// tile of 2^(13-L) rows x 2^L contiguous columns at row stride 2^k, adds 1,
// and writes it back (same addresses).  Sweeps L (segment = 2^L * 8 bytes)
// and k, reports TB/s of algorithmic traffic (16 B/element).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb_stride tools/mb_stride.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

template <int L, int SMEM_KB>
__global__ void __launch_bounds__(256, 2) k_rt(u64* __restrict__ d, int k) {
    extern __shared__ u64 sm[];
    const uint64_t b = blockIdx.x;
    const int mid = k - L;
    const uint64_t base = ((b & ((1ull << mid) - 1ull)) << L) | ((b >> mid) << (k + 13 - L));
    u64 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        const uint64_t off = (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k);
        v[j] = d[base + off];
    }
    if (SMEM_KB > 0) {  // touch smem so the occupancy matches the pass kernels
        sm[threadIdx.x] = v[0];
        __syncthreads();
        v[1] += sm[(threadIdx.x + 1) & 255] & 0;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        const uint64_t off = (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k);
        d[base + off] = v[j] + 1;
    }
}

template <int L>
void run(u64* d, int n, int k) {
    const unsigned grid = 1u << (n - 13);
    const int smem = 66 * 1024;
    cudaFuncSetAttribute(k_rt<L, 66>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) k_rt<L, 66><<<grid, 256, smem>>>(d, k);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_rt<L, 66><<<grid, 256, smem>>>(d, k);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 16.0 * (double)(1ull << n) * reps;
    printf("L=%2d seg=%5d B  k=%2d  %.3f ms  %.2f TB/s  %s\n", L, 8 << L, k, ms / reps, bytes / (ms / 1e3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 32;
    u64* d = nullptr;
    if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
    cudaMemset(d, 0, 8ull << n);
    for (int k : {13, 19}) {
        run<2>(d, n, k);
        run<3>(d, n, k);
        run<4>(d, n, k);
        run<5>(d, n, k);
        run<6>(d, n, k);
        run<8>(d, n, k);
    }
    run<13>(d, n, 13 + 0);  // contiguous tile (k unused when L = 13: mid = 0)
    cudaFree(d);
    return 0;
}
