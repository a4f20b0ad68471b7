// Microbenchmark: the 2-CTA high pass's access pattern with the kernel's own
// LOAD and STORE layouts (CfgHigh14c: round 0 loads with lanes = tile bits
// 0..4, warps 5..7, registers 8..12, rank = bit 13; the store round after
// the DSMEM exchange has lanes {0,1,2,3,8}, warps {9,10,11}, registers
// {4,5,6,7,13} and the rank on tile bit 12), no butterflies.  mb_split.cu
// stores what each thread loaded; here the stores follow the store round,
// as in k_pass / k_pass_split.  The tile's 10 row bits map to any list of
// global bits, so row orders can be compared:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_split2 tools/mb_split2.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__constant__ u64 c_bit[14];      // global offset of tile bit b
__constant__ int c_freebit[40];  // free global bits, ascending (tile id bits)
__constant__ int c_nfree;

__device__ __forceinline__ u64 ld256(const u64* p) {
    u64 v;
    asm volatile("ld.global.L2::256B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ u64 off_of(uint32_t e) {
    u64 o = 0;
#pragma unroll
    for (int b = 0; b < 14; ++b)
        if ((e >> b) & 1u) o += c_bit[b];
    return o;
}

// STORE_MODE 0: stores = the loaded addresses (mb_split); 1: the store round.
template <int STORE_MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) k_walk2(u64* __restrict__ d) {
    extern __shared__ u64 sm[];
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint64_t tile = blockIdx.x >> 1;
    u64 base = 0;
    for (int i = 0; i < c_nfree; ++i) base |= ((tile >> i) & 1ull) << c_freebit[i];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    // round 0: lanes -> tile bits 0..4, warps -> 5..7, registers -> 8..12, rank -> 13
    const uint32_t t0 = lane | (warp << 5) | (rank << 13);
    u64* g = d + base;
    const u64 o0 = off_of(t0);
    u64 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = ld256(g + o0 + off_of((uint32_t)j << 8));
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    sm[threadIdx.x] = v[0];
    __syncthreads();
    v[1] += sm[(threadIdx.x + 1) & 255] & 0;
    if constexpr (STORE_MODE == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) g[o0 + off_of((uint32_t)j << 8)] = v[j] + 1;
    } else {
        // store round: lanes -> {0,1,2,3,8}, warps -> {9,10,11}, regs -> {4,5,6,7,13}, rank -> 12
        const uint32_t t1 = (lane & 15u) | (((lane >> 4) & 1u) << 8) | (warp << 9) | (rank << 12);
        const u64 o1 = off_of(t1);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t e = ((uint32_t)(j & 15) << 4) | ((uint32_t)(j >> 4) << 13);
            g[o1 + off_of(e)] = v[j] + 1;
        }
    }
}

__global__ void k_fill_rand(u64* d, u64 count) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
        u64 z = i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        d[i] = z ^ (z >> 31);
    }
}

template <int M>
static void run(u64* d, int n, std::vector<int> rows, const char* name) {
    std::vector<int> tb;  // tile bit -> global bit (L = 4 columns)
    for (int b = 0; b < 4; ++b) tb.push_back(b);
    for (int r : rows) tb.push_back(r);
    if ((int)tb.size() != 14) { printf("bad tile\n"); return; }
    u64 bit[14];
    for (int b = 0; b < 14; ++b) bit[b] = 1ull << tb[b];
    int freeb[40], nf = 0;
    for (int g = 0; g < n; ++g) {
        bool used = false;
        for (int t : tb) used |= (t == g);
        if (!used) freeb[nf++] = g;
    }
    cudaMemcpyToSymbol(c_bit, bit, sizeof bit);
    cudaMemcpyToSymbol(c_freebit, freeb, sizeof freeb);
    cudaMemcpyToSymbol(c_nfree, &nf, sizeof nf);
    const unsigned grid = 1u << (n - 13);
    const int smem = 66 * 1024;
    cudaFuncSetAttribute(k_walk2<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) k_walk2<M><<<grid, 256, smem>>>(d);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_walk2<M><<<grid, 256, smem>>>(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 16.0 * (double)(1ull << n) * reps;
    printf("%-8s %-40s rows=", M ? "kstore" : "same", name);
    for (int r : rows) printf("%d,", r);
    printf("  %.3f ms  %.2f TB/s  %s\n", ms / reps, bytes / (ms / 1e3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

static std::vector<int> range(int a, int b) {
    std::vector<int> v;
    for (int i = a; i < b; ++i) v.push_back(i);
    return v;
}
static std::vector<int> cat(std::vector<int> a, std::vector<int> b) {
    a.insert(a.end(), b.begin(), b.end());
    return a;
}

int main(int argc, char** argv) {
    const bool rnd = argc > 1 && argv[1][0] == 'r';
    const int n = 34;
    u64* d = nullptr;
    if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
    cudaMemset(d, 0, 8ull << n);
    if (rnd) k_fill_rand<<<148 * 8, 512>>>(d, 1ull << n);
    printf("n=%d data=%s\n", n, rnd ? "random 64-bit" : "zeros");
    struct Case { std::vector<int> rows; const char* name; };
    std::vector<Case> cases = {
        {range(14, 24), "contig k14 (low run)"},
        {range(18, 28), "contig k18 (current pass 3)"},
        {range(24, 34), "contig k24"},
        {cat(range(14, 18), range(28, 34)), "split {14..17}+{28..33} (current pass 2)"},
        {cat(range(28, 34), range(14, 18)), "split high run first, low on 10..13"},
        {cat(cat(range(28, 32), range(14, 18)), range(32, 34)), "split 28..31, 14..17, 32, 33"},
        {cat(cat(range(14, 18), range(32, 34)), range(28, 32)), "split 14..17, 32, 33, 28..31"},
        {cat(range(18, 24), range(30, 34)), "split {18..23}+{30..33}"},
    };
    for (auto& c : cases) {
        run<0>(d, n, c.rows, c.name);
        run<1>(d, n, c.rows, c.name);
    }
    cudaFree(d);
    return 0;
}
