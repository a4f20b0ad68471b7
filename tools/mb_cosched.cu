// Microbenchmark: does co-scheduling CTAs of ADJACENT column groups (a
// thread-block cluster used only for gang scheduling, no DSMEM) help the
// short-segment / large-stride high-pass pattern?  Same tile walk as
// mb_stride.cu (2^(13-L) rows x 2^L columns at row stride 2^k, +1 in place).
//   SYNC = 0: cluster only co-schedules; 1: cluster barrier after the loads
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_cosched tools/mb_cosched.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

template <int L, int SYNC>
__global__ void __launch_bounds__(256, 2) k_rt(u64* __restrict__ d, int k) {
    extern __shared__ u64 sm[];
    const uint64_t b = blockIdx.x;
    const int mid = k - L;
    const uint64_t base = ((b & ((1ull << mid) - 1ull)) << L) | ((b >> mid) << (k + 13 - L));
    u64 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        v[j] = d[base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)];
    }
    if (SYNC) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    sm[threadIdx.x] = v[0];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        d[base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)] = v[j] + 1;
    }
}

template <int L, int SYNC>
void run(u64* d, int n, int k, int cl) {
    const unsigned grid = 1u << (n - 13);
    const int smem = 66 * 1024;
    cudaFuncSetAttribute(k_rt<L, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_rt<L, SYNC>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k_rt<L, SYNC>, d, k);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k_rt<L, SYNC>, d, k);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 16.0 * (double)(1ull << n) * reps;
    printf("L=%d seg=%4dB k=%2d cluster=%d sync=%d  %.2f TB/s  %s\n", L, 8 << L, k, cl, SYNC,
           bytes / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 32;
    u64* d = nullptr;
    if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
    cudaMemset(d, 0, 8ull << n);
    for (int k : {13, 22}) {
        for (int cl : {1, 2, 4, 8}) {
            run<4, 0>(d, n, k, cl);
            if (cl > 1) run<4, 1>(d, n, k, cl);
        }
        for (int cl : {1, 2, 4}) run<3, 0>(d, n, k, cl);
        for (int cl : {1, 2, 4}) run<5, 0>(d, n, k, cl);
    }
    cudaFree(d);
    return 0;
}
