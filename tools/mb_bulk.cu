// Microbenchmark: the high-pass access pattern (2^(13-L) rows x 2^L columns
// at row stride 2^k, in place, +1, no butterflies) fed four ways:
//   A  scalar 8-byte LDG/STG, whole tile in registers, 2 CTAs/SM
//   B  16-byte LDG/STG (pairs of columns), 2 CTAs/SM
//   C  persistent CTAs, S-slot ring of cp.async.bulk row loads (mbarrier
//      complete_tx), registers -> plain STG
//   D  as C, results written back to the slot and stored with
//      cp.async.bulk (bulk_group)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_bulk tools/mb_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ uint64_t tile_base(uint64_t b, int k, int L) {
    const int mid = k - L;
    return ((b & ((1ull << mid) - 1ull)) << L) | ((b >> mid) << (k + 13 - L));
}

template <int L>
__global__ void __launch_bounds__(256, 2) k_a(u64* __restrict__ d, int k) {
    const uint64_t base = tile_base(blockIdx.x, k, L);
    u64 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        v[j] = d[base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)];
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
        d[base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)] = v[j] + 1;
    }
}

template <int L>
__global__ void __launch_bounds__(256, 2) k_b(u64* __restrict__ d, int k) {
    const uint64_t base = tile_base(blockIdx.x, k, L);
    ulonglong2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t e = ((uint32_t)j * 256u + threadIdx.x) * 2u;
        v[j] = *reinterpret_cast<const ulonglong2*>(d + base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k));
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t e = ((uint32_t)j * 256u + threadIdx.x) * 2u;
        ulonglong2 t = v[j];
        t.x += 1;
        t.y += 1;
        *reinterpret_cast<ulonglong2*>(d + base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)) = t;
    }
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(mbar), "r"(parity)
            : "memory");
    }
}

// Warp 0 issues the 2^(13-L) row loads of tile b into slot s.
template <int L>
__device__ __forceinline__ void issue_tile(const u64* d, uint64_t b, int k, uint32_t slot_addr, uint32_t mbar) {
    constexpr int ROWS = 1 << (13 - L);
    constexpr uint32_t SEG = 8u << L;
    const uint32_t lane = threadIdx.x & 31u;
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(8u << 13) : "memory");
    __syncwarp();
    const u64* g = d + tile_base(b, k, L);
    for (int r = lane; r < ROWS; r += 32) {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                slot_addr + (uint32_t)r * SEG),
            "l"(g + ((uint64_t)r << k)), "r"(SEG), "r"(mbar)
            : "memory");
    }
}

template <int L, int S, bool BULK_ST>
__global__ void __launch_bounds__(256, 1) k_c(u64* __restrict__ d, int k, uint64_t ntiles) {
    extern __shared__ __align__(128) u64 sm[];
    constexpr int ROWS = 1 << (13 - L);
    constexpr uint32_t SEG = 8u << L;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t mbase = sbase + S * (8u << 13);
    const uint32_t warp = threadIdx.x >> 5;
    if (threadIdx.x < S)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbase + 8u * threadIdx.x) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (warp == 0)
        for (int s = 0; s < S; ++s)
            if (first + s * step < ntiles) issue_tile<L>(d, first + s * step, k, sbase + s * (8u << 13), mbase + 8u * s);
    uint32_t it = 0;
    for (uint64_t b = first; b < ntiles; b += step, ++it) {
        const uint32_t s = it % S;
        mbar_wait(mbase + 8u * s, (it / S) & 1u);
        u64* slot = sm + (size_t)s * (1u << 13);
        const uint64_t base = tile_base(b, k, L);
        if constexpr (!BULK_ST) {
            u64 v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = slot[j * 256 + threadIdx.x];
            __syncthreads();  // slot consumed
            if (warp == 0 && b + S * step < ntiles)
                issue_tile<L>(d, b + S * step, k, sbase + s * (8u << 13), mbase + 8u * s);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t e = (uint32_t)j * 256u + threadIdx.x;
                d[base + (e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k)] = v[j] + 1;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) slot[j * 256 + threadIdx.x] += 1;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (warp == 0) {
                const uint32_t lane = threadIdx.x & 31u;
                for (int r = lane; r < ROWS; r += 32)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                     d + base + ((uint64_t)r << k)),
                                 "r"(sbase + s * (8u << 13) + (uint32_t)r * SEG), "r"(SEG)
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                // the previous slot's store has read its smem: refill it
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncwarp();
                if (it > 0) {
                    const uint32_t ps = (it - 1) % S;
                    const uint64_t nb = b - step + S * step;
                    if (nb < ntiles) issue_tile<L>(d, nb, k, sbase + ps * (8u << 13), mbase + 8u * ps);
                }
            }
        }
    }
    if constexpr (BULK_ST) {
        if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

template <class F>
float time_it(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    f();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

static int nsm = 148;

template <int L, int S>
void run_l(u64* d, int n, int k) {
    const uint64_t ntiles = 1ull << (n - 13);
    const double gb = 16.0 * (double)(1ull << n) / 1e9;
    float ma = time_it([&] { k_a<L><<<(unsigned)ntiles, 256>>>(d, k); });
    float mb = L >= 1 ? time_it([&] { k_b<L><<<(unsigned)ntiles, 256>>>(d, k); }) : 0.f;
    const int smem = S * (8 << 13) + 64;
    cudaFuncSetAttribute(k_c<L, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_c<L, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float mc = time_it([&] { k_c<L, S, false><<<nsm, 256, smem>>>(d, k, ntiles); });
    float md = time_it([&] { k_c<L, S, true><<<nsm, 256, smem>>>(d, k, ntiles); });
    printf("L=%d seg=%4dB k=%2d S=%d | A %.2f  B %.2f  C %.2f  D %.2f TB/s  (%s)\n", L, 8 << L, k, S, gb / ma,
           gb / mb, gb / mc, gb / md, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int n = 32;
    u64* d = nullptr;
    if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
    cudaMemset(d, 0, 8ull << n);
    for (int k : {13, 22}) {
        run_l<3, 3>(d, n, k);
        run_l<4, 3>(d, n, k);
        run_l<5, 3>(d, n, k);
        run_l<8, 3>(d, n, k);
    }
    run_l<4, 2>(d, n, 13);
    // correctness of the ring variants: every element incremented once per launch
    cudaMemset(d, 0, 8ull << n);
    const uint64_t ntiles = 1ull << (n - 13);
    const int smem = 3 * (8 << 13) + 64;
    k_c<4, 3, false><<<nsm, 256, smem>>>(d, 13, ntiles);
    k_c<4, 3, true><<<nsm, 256, smem>>>(d, 13, ntiles);
    k_a<4><<<(unsigned)ntiles, 256>>>(d, 13);
    u64 h[4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    u64 t;
    cudaMemcpy(&t, d + (1ull << n) - 1, 8, cudaMemcpyDeviceToHost);
    printf("check %llu %llu %llu (want 3) %s\n", h[0], h[3], t, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    return 0;
}
