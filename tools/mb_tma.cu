// Microbenchmark: the high-pass access pattern (2^(13-L) rows x 2^L columns
// at row stride 2^k, in place, +1, no butterflies) fed by TENSOR-map TMA:
// persistent CTAs (one per SM), an S-slot ring of 64 KB tiles, each tile
// fetched as 2D boxes of {2^L columns x 256 rows} (one instruction per 256
// rows), completion on an mbarrier.
//   T1: TMA loads, registers, plain STG stores
//   T2: TMA loads, +1 in shared memory, TMA tensor stores (bulk_group)
// Compare with mb_bulk.cu A/B (LDG/STG, whole tile in registers, 2 CTAs/SM).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_tma tools/mb_tma.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

typedef unsigned long long u64;

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

// tile b: column group c = b % groups, row block rb = b / groups (2^(13-L) rows)
template <int L>
__device__ __forceinline__ void issue_tile(const CUtensorMap* tm, uint64_t b, int groups_log2, uint32_t slot,
                                           uint32_t mbar) {
    constexpr int ROWS = 1 << (13 - L);
    const int c = (int)(b & ((1ull << groups_log2) - 1));
    const int rb = (int)(b >> groups_log2);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(8u << 13) : "memory");
#pragma unroll
    for (int h = 0; h < ROWS / 256; ++h) {
        const int row0 = rb * ROWS + h * 256;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];" ::"r"(slot + (uint32_t)h * 256u * (8u << L)),
            "l"(tm), "r"(0), "r"(c), "r"(row0), "r"(mbar)
            : "memory");
    }
}

template <int L>
__device__ __forceinline__ void store_tile(const CUtensorMap* tm, uint64_t b, int groups_log2, uint32_t slot) {
    constexpr int ROWS = 1 << (13 - L);
    const int c = (int)(b & ((1ull << groups_log2) - 1));
    const int rb = (int)(b >> groups_log2);
#pragma unroll
    for (int h = 0; h < ROWS / 256; ++h) {
        const int row0 = rb * ROWS + h * 256;
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
                     "r"(0), "r"(c), "r"(row0), "r"(slot + (uint32_t)h * 256u * (8u << L))
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int L, int S, bool TMA_ST>
__global__ void __launch_bounds__(256, 1)
    k_tma(const __grid_constant__ CUtensorMap tm, u64* __restrict__ d, int k, int groups_log2, uint64_t ntiles) {
    extern __shared__ __align__(1024) u64 sm[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t mbase = sbase + S * (8u << 13);
    if (threadIdx.x < S)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbase + 8u * threadIdx.x) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const uint64_t first = blockIdx.x, step = gridDim.x;
    if (threadIdx.x == 0)
        for (int s = 0; s < S; ++s)
            if (first + s * step < ntiles)
                issue_tile<L>(&tm, first + s * step, groups_log2, sbase + s * (8u << 13), mbase + 8u * s);
    uint32_t it = 0;
    for (uint64_t b = first; b < ntiles; b += step, ++it) {
        const uint32_t s = it % S;
        mbar_wait(mbase + 8u * s, (it / S) & 1u);
        u64* slot = sm + (size_t)s * (1u << 13);
        if constexpr (!TMA_ST) {
            const int c = (int)(b & ((1ull << groups_log2) - 1));
            const uint64_t rb = b >> groups_log2;
            const uint64_t base = ((uint64_t)c << L) + ((rb << (13 - L)) << k);
            u64 v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = slot[j * 256 + threadIdx.x];
            __syncthreads();  // slot consumed
            if (threadIdx.x == 0 && b + S * step < ntiles)
                issue_tile<L>(&tm, b + S * step, groups_log2, sbase + s * (8u << 13), mbase + 8u * s);
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
            if (threadIdx.x == 0) {
                store_tile<L>(&tm, b, groups_log2, sbase + s * (8u << 13));
                // the previous tile's store has read its slot: refill that slot
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                if (it > 0) {
                    const uint32_t ps = (it - 1) % S;
                    const uint64_t nb = b - step + S * step;
                    if (nb < ntiles) issue_tile<L>(&tm, nb, groups_log2, sbase + ps * (8u << 13), mbase + 8u * ps);
                }
            }
        }
    }
    if constexpr (TMA_ST) {
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

template <int L>
CUtensorMap make_map(u64* d, int n, int k) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)1 << L, (cuuint64_t)1 << (k - L), (cuuint64_t)1 << (n - k)};
    cuuint64_t strides[2] = {(cuuint64_t)8 << L, (cuuint64_t)8 << k};
    cuuint32_t box[3] = {1u << L, 1u, 256u};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, d, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return tm;
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

template <int L, int S>
void run(u64* d, int n, int k, int nsm) {
    const uint64_t ntiles = 1ull << (n - 13);
    const double gb = 16.0 * (double)(1ull << n) / 1e9;
    CUtensorMap tm = make_map<L>(d, n, k);
    const int smem = S * (8 << 13) + 64;
    cudaFuncSetAttribute(k_tma<L, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_tma<L, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float m1 = time_it([&] { k_tma<L, S, false><<<nsm, 256, smem>>>(tm, d, k, k - L, ntiles); });
    float m2 = time_it([&] { k_tma<L, S, true><<<nsm, 256, smem>>>(tm, d, k, k - L, ntiles); });
    printf("L=%d seg=%4dB k=%2d S=%d | T1 (TMA ld, STG) %.2f  T2 (TMA ld+st) %.2f TB/s  (%s)\n", L, 8 << L, k, S,
           gb / m1, gb / m2, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    if (!encode) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int n = 32;
    u64* d = nullptr;
    if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
    cudaMemset(d, 0, 8ull << n);
    for (int k : {13, 22}) {
        run<3, 3>(d, n, k, nsm);
        run<4, 3>(d, n, k, nsm);
        run<5, 3>(d, n, k, nsm);
    }
    // correctness: each launch adds 1 to every element
    cudaMemset(d, 0, 8ull << n);
    CUtensorMap tm = make_map<4>(d, n, 13);
    const int smem = 3 * (8 << 13) + 64;
    k_tma<4, 3, false><<<nsm, 256, smem>>>(tm, d, 13, 9, 1ull << (n - 13));
    k_tma<4, 3, true><<<nsm, 256, smem>>>(tm, d, 13, 9, 1ull << (n - 13));
    u64 h[3];
    cudaMemcpy(&h[0], d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&h[1], d + 12345677, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&h[2], d + (1ull << n) - 1, 8, cudaMemcpyDeviceToHost);
    printf("check %llu %llu %llu (want 2) %s\n", h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    return 0;
}
