// Microbenchmark: HBM rate of a pass whose stage rows are NOT one run of
// consecutive global bits.  Same walk as the 10/9-stage 2-CTA passes (a 2^14
// tile on a cluster of 2, cluster rank = top tile bit, 256 threads x 32
// int64 per CTA, 2 CTAs/SM, L2::256B loads), but the tile's global bits are
// an arbitrary set: columns [0, L) plus any row bits.  Tile ids fill the
// remaining global bits in ascending order (column groups first, as
// tile_base does).  Load -> +1 -> store, no butterflies: the access-pattern
// ceiling of a plan that uses split row sets (e.g. rows {13,14,15} u [26,32)).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/mb_split tools/mb_split.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__constant__ u64 c_joff[32];     // offset of register index j (tile bits 8..12)
__constant__ u64 c_rankoff[2];   // offset of the cluster rank (tile bit 13)
__constant__ u64 c_tidmask[8];   // global bit of tile bits 0..7 (thread index)
__constant__ int c_freebit[40];  // free global bits, ascending (tile id bits)
__constant__ int c_nfree;

__device__ __forceinline__ u64 ld256(const u64* p) {
    u64 v;
    asm volatile("ld.global.L2::256B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2) k_walk(u64* __restrict__ d) {
    extern __shared__ u64 sm[];
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint64_t tile = blockIdx.x >> 1;
    u64 base = 0;
    for (int i = 0; i < c_nfree; ++i) base |= ((tile >> i) & 1ull) << c_freebit[i];
    u64 toff = c_rankoff[rank];
#pragma unroll
    for (int b = 0; b < 8; ++b) toff += ((threadIdx.x >> b) & 1u) ? c_tidmask[b] : 0ull;
    u64* g = d + base + toff;
    u64 v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = ld256(g + c_joff[j]);
    sm[threadIdx.x] = v[0];  // occupancy like the pass kernels (66 KB smem)
    __syncthreads();
    v[1] += sm[(threadIdx.x + 1) & 255] & 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) g[c_joff[j]] = v[j] + 1;
}

// Fill with high-entropy 64-bit values (SplitMix64 of the index): the
// config-5 passes see such data, the zero-filled walk does not.
__global__ void k_fill_rand(u64* d, u64 count) {
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
        u64 z = i * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        d[i] = z ^ (z >> 31);
    }
}

// rows: the 14 - L global row bits, in tile-bit order (the last one is the
// cluster rank).
static void run(u64* d, int n, int L, std::vector<int> rows, const char* name) {
    std::vector<int> tb;  // tile bit -> global bit
    for (int b = 0; b < L; ++b) tb.push_back(b);
    for (int r : rows) tb.push_back(r);
    if ((int)tb.size() != 14) { printf("bad tile\n"); return; }
    u64 joff[32], rankoff[2] = {0, 1ull << tb[13]}, tidm[8];
    for (int b = 0; b < 8; ++b) tidm[b] = 1ull << tb[b];
    for (int j = 0; j < 32; ++j) {
        joff[j] = 0;
        for (int i = 0; i < 5; ++i)
            if ((j >> i) & 1) joff[j] |= 1ull << tb[8 + i];
    }
    int freeb[40], nf = 0;
    for (int g = 0; g < n; ++g) {
        bool used = false;
        for (int t : tb) used |= (t == g);
        if (!used) freeb[nf++] = g;
    }
    cudaMemcpyToSymbol(c_joff, joff, sizeof joff);
    cudaMemcpyToSymbol(c_rankoff, rankoff, sizeof rankoff);
    cudaMemcpyToSymbol(c_tidmask, tidm, sizeof tidm);
    cudaMemcpyToSymbol(c_freebit, freeb, sizeof freeb);
    cudaMemcpyToSymbol(c_nfree, &nf, sizeof nf);
    const unsigned grid = 1u << (n - 13);
    const int smem = 66 * 1024;
    cudaFuncSetAttribute(k_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) k_walk<<<grid, 256, smem>>>(d);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_walk<<<grid, 256, smem>>>(d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = 16.0 * (double)(1ull << n) * reps;
    printf("%-34s L=%d rows=", name, L);
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
    // argv[1] == "rand": high-entropy data (else zeros, incremented by each walk)
    const bool rnd = argc > 1 && argv[1][0] == 'r' && argv[1][1] != '1';
    if (argc > 1 && !strcmp(argv[1], "r11")) {
        // 11-row passes on a 2^14 tile (3 column bits, 64-byte segments): would
        // let n = 34 run 13 + 11 + 10 instead of 14 + 10 + 10.
        const int n = 34;
        u64* d = nullptr;
        if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
        cudaMemset(d, 0, 8ull << n);
        printf("n=%d data=zeros, 11-row walks\n", n);
        run(d, n, 3, range(13, 24), "contig r11 k13");
        run(d, n, 3, cat(range(13, 18), range(28, 34)), "split r11 {13..17}+{28..33}");
        run(d, n, 3, cat(range(13, 19), range(29, 34)), "split r11 {13..18}+{29..33}");
        run(d, n, 3, cat(range(13, 20), range(30, 34)), "split r11 {13..19}+{30..33}");
        run(d, n, 3, cat(range(13, 21), range(31, 34)), "split r11 {13..20}+{31..33}");
        run(d, n, 4, range(19, 29), "contig r10 k19");
        run(d, n, 4, cat(range(14, 18), range(28, 34)), "split r10 {14..17}+{28..33} (current)");
        cudaFree(d);
        return 0;
    }
    for (int n : {32, 34}) {
        u64* d = nullptr;
        if (cudaMalloc(&d, 8ull << n) != cudaSuccess) return 1;
        cudaMemset(d, 0, 8ull << n);
        if (rnd) k_fill_rand<<<148 * 8, 512>>>(d, 1ull << n);
        printf("n=%d data=%s\n", n, rnd ? "random 64-bit" : "zeros");
        if (n == 32) {
            run(d, n, 4, range(13, 23), "contig r10 k13 (current pass 2)");
            run(d, n, 4, range(14, 24), "contig r10 k14");
            run(d, n, 4, range(16, 26), "contig r10 k16");
            run(d, n, 5, range(23, 32), "contig r9 k23 (current pass 3)");
            run(d, n, 5, cat(range(13, 16), range(26, 32)), "split r9 {13..15}+{26..31}");
            run(d, n, 5, cat(range(26, 32), range(13, 16)), "split r9 rank on 15");
            run(d, n, 4, cat(range(13, 16), range(25, 32)), "split r10 {13..15}+{25..31}");
            run(d, n, 5, cat(range(13, 14), range(24, 32)), "split r9 {13}+{24..31}");
        } else {
            run(d, n, 4, range(14, 24), "contig r10 k14 (current pass 2)");
            run(d, n, 4, range(24, 34), "contig r10 k24 (current pass 3)");
            run(d, n, 4, range(18, 28), "contig r10 k18");
            run(d, n, 4, cat(range(14, 18), range(28, 34)), "split r10 {14..17}+{28..33}");
            run(d, n, 4, cat(range(28, 34), range(14, 18)), "split r10 rank on 17");
            run(d, n, 4, cat(range(14, 16), range(26, 34)), "split r10 {14,15}+{26..33}");
        }
        cudaFree(d);
    }
    return 0;
}
