// bw_kernels32.cuh -- the int32 register engine of the compact plan.
//
// The compact in-place plan (bw_abi.cu, bw_fwht_i64_compact) keeps the
// signal as int32 inside its own buffer between the first high pass and the
// low pass.  The int64 engine (bw_kernels.cuh) holds 2^13 elements per CTA,
// so on int32 data it moves half the bytes per tile, and a pass's time is
// set by its load latency and per-tile machinery, not by its bytes
// (DESIGN.md section 5).  This engine holds 2^14 int32 per CTA (256 threads
// x 64 registers, 64 KiB of shared memory, two CTAs per SM): the same bytes
// in flight per tile as the int64 engine, so an int32 pass should take the
// time of its bytes.
//
//   k32_first<L, MODE>: the plan's first pass, natural int64 -> int32 in
//     place (8 or 9 rows), with the input test of the unknown-bound case
//     (MODE = FIRST_CHECK); k32_restore<L> undoes it on the tiles it wrote.
//   k32_high<L>: int32 -> int32 high pass, r = 14 - L = 6..9 stage rows of the
//     compact layout (2^L contiguous int32 columns, rows at slot stride
//     2^(k+1)); one CTA per tile, two rounds joined by one shared-memory
//     transpose.
//   k32_low<EX>: int32 -> int64 low pass (stages 0..13 of every 2^14 block),
//     reading the block's int32 half and writing the natural int64 block.
//     Rounds 0 and 1 stage 10 bits in int32; round 2 runs as two sub-rounds
//     of 2^13 elements (32 per thread) that widen to int64 and stage the
//     last 4 bits (10..13) in int64 registers, then store 16-byte pairs.
//     EX: the threshold extraction (|W| >= tau) on the final registers.
//
// Exactness: the plan admits only |x| <= (2^31 - 1) >> (n - 4) (bw_abi.cu
// compact_plan), so every int32 intermediate -- all stages but the last
// four -- is the exact value and the wrapping uint32 add/sub below equals it.
//
// Layout tables use the nibble packing of bw_layouts.h: round RD assigns
// every virtual tile bit (0..13) to a register bit (6, or 5 in the low
// pass's sub-rounds), a lane bit (5) or a warp bit (3); butterflies run on
// register bits.  Shared-memory slots are a linear XOR swizzle of the tile
// index, chosen so that every 4/8/16-byte access phase of every round is
// conflict-free (bw_plan_check_compact verifies every round of every config).
#pragma once
#include <stdint.h>

#include "bw_kernels.cuh"
#include "bw_layouts.h"

namespace bw {
namespace w32 {

typedef uint32_t u32;
constexpr int kBits = 14;  // elements per CTA tile
constexpr int kNT = 256;   // threads per CTA
constexpr int kE = 64;     // int32 registers per thread
constexpr int kSmemBytes = 4 << kBits;

// Low pass over stages 0..13, int32 compact source -> int64 natural.
// Virtual bit b = index bit i_b of the block.
//   round 0: reg {0,1,6,7,8,9}    lane {2,3,13,4,5}  warp {10,11,12}  stages 0,1,6..9   (16-byte loads)
//   round 1: reg {0,1,2,3,4,5}    lane {6..10}       warp {11,12,13}  stages 2..5
//   round 2: reg {0,10,11,12,13}  lane {1..5}        warp {6,7,8}     stages 10..13 in int64,
//            sub-round bit 9 (two halves of 32 values per thread), 16-byte int64 stores
// Source slot of the compact layout (bw_abi.cu compact_layout, w = 14):
// i0..i3 -> 0..3, i13 -> 4, i4..i12 -> 5..13.
struct CfgLowW {
    static constexpr int NR = 3;
    static constexpr int SUB = 9;
    BW_HD static constexpr int nreg(int rd) { return rd == 2 ? 5 : 6; }
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(rd == 0 ? 0x987610ull : rd == 1 ? 0x543210ull : 0xDCBA0ull, i);
    }
    BW_HD static constexpr int lane(int rd, int i) {
        return nib(rd == 0 ? 0x54D32ull : rd == 1 ? 0xA9876ull : 0x54321ull, i);
    }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0xCBAull : rd == 1 ? 0xDCBull : 0x876ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x3C3u : rd == 1 ? 0x3Cu : 0x3C00u; }
    // slot bits 2, 3, 4 ^= e6, e7, e8 ^ e13
    BW_HD static constexpr uint32_t slot(uint32_t e) { return e ^ ((e >> 4) & 0x1Cu) ^ ((e >> 9) & 0x10u); }
    BW_HD static constexpr uint32_t src_off(uint32_t e) {
        return (e & 0xFu) | (((e >> 13) & 1u) << 4) | (((e >> 4) & 0x1FFu) << 5);
    }
};

// High pass, r = 14 - L rows: virtual bits 0..L-1 are the columns (slot bits
// 0..L-1 of the compact layout), L..13 the rows.
//   L = 5 (9 rows): round 0 reg {0,5..9}     lane {1,2,3,4,10} warp {11,12,13} stages 5..9  (8-byte loads)
//                   round 1 reg {0,1,10..13} lane {2..6}       warp {7,8,9}    stages 10..13 (16-byte stores)
//   L = 6 (8 rows): round 0 reg {0,6..10}    lane {1..5}       warp {11,12,13} stages 6..10
//                   round 1 reg {0,1,11,12,13,6} lane {2,3,4,5,7} warp {8,9,10} stages 11..13
//   L = 7 (7 rows): round 0 reg {0,7..11}    lane {1..5}       warp {6,12,13}  stages 7..11
//                   round 1 reg {0,1,12,13,7,8} lane {2..6}    warp {9,10,11}  stages 12, 13
//   L = 8 (6 rows): round 0 reg {0,8..12}    lane {1..5}       warp {6,7,13}   stages 8..12
//                   round 1 reg {0,1,13,8,9,10} lane {2..6}    warp {7,11,12}  stage 13
// (L = 7, 8: second passes only, as 8 rows then 7 / 6 at n = 29 / 28.)
template <int L>
struct CfgHighW {
    static_assert(L >= 5 && L <= 8, "int32 high passes of 6 to 9 rows");
    static constexpr int NR = 2;
    BW_HD static constexpr int nreg(int) { return 6; }
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(L == 5   ? (rd == 0 ? 0x987650ull : 0xDCBA10ull)
                   : L == 6 ? (rd == 0 ? 0xA98760ull : 0x6DCB10ull)
                   : L == 7 ? (rd == 0 ? 0xBA9870ull : 0x87DC10ull)
                            : (rd == 0 ? 0xCBA980ull : 0xA98D10ull),
                   i);
    }
    BW_HD static constexpr int lane(int rd, int i) {
        return nib(L == 5   ? (rd == 0 ? 0xA4321ull : 0x65432ull)
                   : L == 6 ? (rd == 0 ? 0x54321ull : 0x75432ull)
                            : (rd == 0 ? 0x54321ull : 0x65432ull),
                   i);
    }
    BW_HD static constexpr int warp(int rd, int i) {
        return nib(L == 5   ? (rd == 0 ? 0xDCBull : 0x987ull)
                   : L == 6 ? (rd == 0 ? 0xDCBull : 0xA98ull)
                   : L == 7 ? (rd == 0 ? 0xDC6ull : 0xBA9ull)
                            : (rd == 0 ? 0xD76ull : 0xCB7ull),
                   i);
    }
    BW_HD static constexpr uint32_t stage(int rd) {
        return L == 5   ? (rd == 0 ? 0x3E0u : 0x3C00u)
               : L == 6 ? (rd == 0 ? 0x7C0u : 0x3800u)
               : L == 7 ? (rd == 0 ? 0xF80u : 0x3000u)
                        : (rd == 0 ? 0x1F00u : 0x2000u);
    }
    BW_HD static constexpr uint32_t slot(uint32_t e) { return e; }
};

// Tile index bits of register index j in round RD.
template <class C, int RD>
BW_HD constexpr uint32_t reg_part(int j) {
    uint32_t e = 0;
    for (int i = 0; i < C::nreg(RD); ++i)
        if ((j >> i) & 1) e |= 1u << C::reg(RD, i);
    return e;
}

template <class C, int RD>
BW_HD inline uint32_t thread_part(uint32_t lane, uint32_t warp) {
    uint32_t e = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 5; ++i) e |= ((lane >> i) & 1u) << C::lane(RD, i);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 3; ++i) e |= ((warp >> i) & 1u) << C::warp(RD, i);
    return e;
}

// Elements per shared-memory / global access of round RD: registers 0 and 1
// on tile bits 0 and 1 give 4 consecutive int32, register 0 on bit 0 a pair.
template <class C, int RD>
BW_HD constexpr int vec() {
    return C::reg(RD, 0) != 0 ? 1 : (C::nreg(RD) > 1 && C::reg(RD, 1) == 1) ? 4 : 2;
}

// Element offset of tile index e in a high pass's tile (kk = k + 1: the
// compact layout moves index bits >= 14 up by one slot bit).
template <int L>
BW_HD inline uint64_t high_off(uint32_t e, int kk) {
    return (uint64_t)(e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << kk);
}

// Slot of element 0 of tile t: the free slot bits [L, 14), [15, kk),
// [kk + 14 - L, ...) take the tile id's bits in ascending order, so
// neighbouring CTAs run neighbouring column groups.
template <int L>
BW_HD inline uint64_t high_tile_base(uint64_t t, int kk) {
    constexpr int m1 = kBits - L;
    const int m2 = kk - (kBits + 1);
    const uint64_t lo = t & ((1ull << m1) - 1ull);
    const uint64_t mid = (t >> m1) & ((1ull << m2) - 1ull);
    const uint64_t hi = t >> (m1 + m2);
    return (lo << L) | (mid << (kBits + 1)) | (hi << (kk + kBits - L));
}

#if defined(__CUDACC__)
template <class C, int RD>
__device__ __forceinline__ void stages32(u32 (&v)[kE]) {
#pragma unroll
    for (int i = 0; i < C::nreg(RD); ++i) {
        if ((C::stage(RD) >> C::reg(RD, i)) & 1u) {
#pragma unroll
            for (int j = 0; j < kE; ++j) {
                if (!((j >> i) & 1)) {
                    const u32 a = v[j], b = v[j | (1 << i)];
                    v[j] = a + b;
                    v[j | (1 << i)] = a - b;
                }
            }
        }
    }
}

template <class C, int RD>
__device__ __forceinline__ void smem_store32(const u32 (&v)[kE], u32* sm, uint32_t tp) {
    constexpr int V = vec<C, RD>();
    const uint32_t st = C::slot(tp);
#pragma unroll
    for (int j = 0; j < kE; j += V) {
        u32* p = sm + (st ^ C::slot(reg_part<C, RD>(j)));
        if constexpr (V == 4) *reinterpret_cast<uint4*>(p) = make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        else if constexpr (V == 2) *reinterpret_cast<uint2*>(p) = make_uint2(v[j], v[j + 1]);
        else *p = v[j];
    }
}

template <class C, int RD>
__device__ __forceinline__ void smem_load32(u32 (&v)[kE], const u32* sm, uint32_t tp) {
    constexpr int V = vec<C, RD>();
    const uint32_t st = C::slot(tp);
#pragma unroll
    for (int j = 0; j < kE; j += V) {
        const u32* p = sm + (st ^ C::slot(reg_part<C, RD>(j)));
        if constexpr (V == 4) {
            const uint4 t = *reinterpret_cast<const uint4*>(p);
            v[j] = t.x;
            v[j + 1] = t.y;
            v[j + 2] = t.z;
            v[j + 3] = t.w;
        } else if constexpr (V == 2) {
            const uint2 t = *reinterpret_cast<const uint2*>(p);
            v[j] = t.x;
            v[j + 1] = t.y;
        } else {
            v[j] = *p;
        }
    }
}

__device__ __forceinline__ uint4 ld4(const u32* p) {
    uint4 t;
    asm volatile("ld.global.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                 : "l"(p));
    return t;
}
__device__ __forceinline__ uint2 ld2(const u32* p) {
    uint2 t;
    asm volatile("ld.global.L2::256B.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "l"(p));
    return t;
}
__device__ __forceinline__ u32 ld1(const u32* p) {
    u32 t;
    asm volatile("ld.global.L2::256B.u32 %0, [%1];" : "=r"(t) : "l"(p));
    return t;
}

// rounds 0 and 1 of a high pass on registers v (loaded in round 0's layout),
// ending with the int32 stores into the compact layout
// CHECK (k32_first's input test): the barrier between the rounds also
// carries the tile's verdict -- no global store precedes it -- so a tile with
// a bad input, or one that saw the abort word, stops there having written
// nothing; the others flag themselves and store.
// PRE_SYNC (k32_first with half its loads landing in shared memory): one
// more barrier after round 0's stages, before the transpose overwrites the
// landing slots other threads may still be reading.
template <int L, bool CHECK = false, bool PRE_SYNC = false, class C = CfgHighW<L>>
__device__ __forceinline__ void high_rounds_store(u32 (&v)[kE], u32* sm32, u32* dst, uint64_t base, int kk, uint32_t lane,
                                                  uint32_t warp, bool bad = false, unsigned* tileflag = nullptr,
                                                  unsigned* abort = nullptr) {
    stages32<C, 0>(v);
    if constexpr (PRE_SYNC) {
        BW_STRESS(68);
        __syncthreads();
    }
    BW_STRESS(60);
    smem_store32<C, 0>(v, sm32, thread_part<C, 0>(lane, warp));
    BW_STRESS(61);
    if constexpr (CHECK) {
        if (__syncthreads_or(bad)) {
            if (threadIdx.x == 0) atomicExch(abort, 1u);
            return;
        }
        if (threadIdx.x == 0) tileflag[blockIdx.x] = 1u;
    } else {
        __syncthreads();
    }
    const uint32_t tp = thread_part<C, 1>(lane, warp);
    smem_load32<C, 1>(v, sm32, tp);
    stages32<C, 1>(v);
    u32* p = dst + base + high_off<L>(tp, kk);
    constexpr int V = vec<C, 1>();
#pragma unroll
    for (int j = 0; j < kE; j += V) {
        u32* q = p + high_off<L>(reg_part<C, 1>(j), kk);
        if constexpr (V == 4) *reinterpret_cast<uint4*>(q) = make_uint4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        else if constexpr (V == 2) *reinterpret_cast<uint2*>(q) = make_uint2(v[j], v[j + 1]);
        else *q = v[j];
    }
}

// int32 -> int32 high pass over rows [k, k + 14 - L) of the compact layout.
// src / dst: the int32 view of the signal, offset by the read / write half.
template <int L, int MINB = 2, class C = CfgHighW<L>>
__global__ void __launch_bounds__(kNT, MINB) k32_high(const u32* __restrict__ src, u32* __restrict__ dst, int k) {
    extern __shared__ __align__(16) u32 sm32[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const int kk = k + 1;
    const uint64_t base = high_tile_base<L>(blockIdx.x, kk);
    u32 v[kE];
    {
        const uint32_t tp = thread_part<C, 0>(lane, warp);
        const u32* p = src + base + high_off<L>(tp, kk);
        constexpr int V = vec<C, 0>();
#pragma unroll
        for (int j = 0; j < kE; j += V) {
            const u32* q = p + high_off<L>(reg_part<C, 0>(j), kk);
            if constexpr (V == 4) {
                const uint4 t = ld4(q);
                v[j] = t.x;
                v[j + 1] = t.y;
                v[j + 2] = t.z;
                v[j + 3] = t.w;
            } else if constexpr (V == 2) {
                const uint2 t = ld2(q);
                v[j] = t.x;
                v[j + 1] = t.y;
            } else {
                v[j] = ld1(q);
            }
        }
    }
    high_rounds_store<L, false, false, C>(v, sm32, dst, base, kk, lane, warp);
}

// int32 -> int32 pass of R = 1..4 stage rows in registers only (no shared
// memory, no barrier): the third high pass of the n = 33 / 34 plans.  Every
// thread holds 4 consecutive slots (16-byte accesses) of 2^R rows; a warp
// covers 512 contiguous bytes of each row.  u = the thread's linear index
// over the half's slots without the row bits; src / dst: the read / write
// half (never in place).
template <int R>
BW_HD inline uint64_t reg_slot_base(uint64_t u, int kk) {
    const uint64_t lo = u & ((1ull << kBits) - 1ull);                      // slot bits 0..13
    const uint64_t mid = (u >> kBits) & ((1ull << (kk - (kBits + 1))) - 1ull);  // slot bits 15..kk-1
    const uint64_t hi = u >> (kk - 1);                                      // above the rows
    return lo | (mid << (kBits + 1)) | (hi << (kk + R));
}

template <int R>
__global__ void __launch_bounds__(kNT) k32_reg(const u32* __restrict__ src, u32* __restrict__ dst, int k) {
    static_assert(R >= 1 && R <= 4, "1 to 4 rows in registers");
    constexpr int NR = 1 << R;
    const int kk = k + 1;
    const uint64_t base = reg_slot_base<R>(((uint64_t)blockIdx.x * kNT + threadIdx.x) * 4u, kk);
    uint4 v[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) v[r] = ld4(src + base + ((uint64_t)r << kk));
#pragma unroll
    for (int i = 0; i < R; ++i) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (!((r >> i) & 1)) {
                const uint4 a = v[r], b = v[r | (1 << i)];
                v[r] = make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
                v[r | (1 << i)] = make_uint4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) *reinterpret_cast<uint4*>(dst + base + ((uint64_t)r << kk)) = v[r];
}

// ---------------------------------------------------------------------------
// The plan's FIRST pass on this engine: natural int64 -> int32 compact, the
// same tile, rounds and stores as k32_high<L> (k = 14: rows 14 .. 14 + r).
// The tile's columns are index bits {0,1,2,3,13} (L = 6: and 4), so every
// int32 slot it writes lies inside the int64 bytes it read itself (in place;
// bw_plan_check_compact runs these exact address functions).
//
// Loads: 16-byte int64 pairs, narrowed as they arrive, in four groups of 16
// values so that at most half of the 128 registers hold raw int64 data.
// FIRST_CHECK: every input is tested against |x| <= lim (the high word is the
// sign extension of the low word, and |low| <= lim).  A tile that finds the
// abort word set, or a bad input, stores nothing (the verdict rides on the
// barrier between the two rounds); else it sets tileflag[tile] and stores.
// So after the pass every tile either holds its int32 output or its
// untouched int64 input, and the flags say which (k32_restore).
// ---------------------------------------------------------------------------
enum { FIRST_PLAIN = 0, FIRST_CHECK = 1 };

// natural int64 offset of tile index e (rows at index bits k ..)
template <int L>
BW_HD inline uint64_t first_off(uint32_t e, int k) {
    return (uint64_t)(e & 15u) | ((uint64_t)((e >> 4) & 1u) << 13) |
           ((uint64_t)((e >> 5) & ((1u << (L - 5)) - 1u)) << 4) | ((uint64_t)(e >> L) << k);
}
// natural index of a tile's element 0 from its compact slot base: slot bits
// 5..13 are index bits 4..12, slot bits >= 15 index bits >= 14
BW_HD inline uint64_t first_base(uint64_t slot_base) {
    return (((slot_base >> 5) & 0x1FFull) << 4) | ((slot_base >> 15) << 14);
}

__device__ __forceinline__ ulonglong2 ld2x64(const unsigned long long* p) {
    ulonglong2 t;
    asm volatile("ld.global.L2::256B.v2.u64 {%0, %1}, [%2];" : "=l"(t.x), "=l"(t.y) : "l"(p));
    return t;
}

// FIRST_CHECK's evidence against a pair of inputs.  CHK 0: per value, the
// high word against the low word's sign extension and |low| (4 operations
// per value on two serial chains).  CHK 1: y = x + lim in 64 bits; |x| <= lim
// iff y <= 2 lim, i.e. high(y) == 0 and low(y) <= 2 lim (lim < 2^31): OR of
// the high words, max of the low words, on four independent accumulators.
struct FirstAcc {
    u32 hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
};
template <int MODE, int CHK>
__device__ __forceinline__ void first_test(const ulonglong2& t, int q, u32 lim, FirstAcc& acc) {
    if constexpr (MODE == FIRST_CHECK) {
        if constexpr (CHK == 0) {
            const int a = (int)(u32)t.x, b = (int)(u32)t.y;
            acc.hi[0] |= ((u32)(t.x >> 32) ^ (u32)(a >> 31)) | ((u32)(t.y >> 32) ^ (u32)(b >> 31));
            acc.lo[0] |= (u32)__builtin_abs(a) | (u32)__builtin_abs(b);  // abs(INT_MIN) = 2^31 as unsigned: rejected
        } else {
            const unsigned long long y0 = t.x + lim, y1 = t.y + lim;
            acc.hi[q & 3] |= (u32)(y0 >> 32) | (u32)(y1 >> 32);
            acc.lo[q & 3] = max(acc.lo[q & 3], max((u32)y0, (u32)y1));
        }
    }
}
template <int CHK>
__device__ __forceinline__ bool first_bad(const FirstAcc& acc, u32 lim) {
    const u32 hi = acc.hi[0] | acc.hi[1] | acc.hi[2] | acc.hi[3];
    const u32 lo = max(max(acc.lo[0], acc.lo[1]), max(acc.lo[2], acc.lo[3]));
    return hi != 0u || lo > (CHK == 0 ? lim : 2u * lim);
}

// VAR (measured variants of the load phase, tools/mb_first32.cu):
//   0: all 32 pair loads into registers, narrowed in four groups;
//   1: as 0 with the abort word read before them;
//   2: registers 32..63 land in the CTA's (still unused) shared memory through
//      cp.async, registers 0..31 through plain loads: the whole tile is in
//      flight at once with 64 instead of 128 registers of raw data, so the
//      checked pass (which needs the high words) no longer splits its loads;
//   3: as 2 with the biased-add test (CHK 1);
//   4: as 3, and a tile that finds the abort word set returns before loading (one more barrier,
//      behind the abort word's load).
// n = 32, 12 B/point: plain 8.02 ms in every variant; checked 9.7 (0, 1),
// 8.6 (2), 8.13 (3), 8.00 (4: the barrier at the start costs nothing, the
// warps then issue their loads together) -- profiles/r02_compact/mb_first32*.log.
constexpr int kFirstVar = 4;

template <int L, int MODE, int VAR = kFirstVar>
__global__ void __launch_bounds__(kNT, 2)
    k32_first(const unsigned long long* __restrict__ src, u32* __restrict__ dst, int k, u32 lim, unsigned* tileflag,
              unsigned* abort) {
    using C = CfgHighW<L>;
    static_assert(vec<C, 0>() == 2, "int64 pairs in round 0");
    constexpr int CHK = VAR >= 3 ? 1 : 0;
    constexpr bool LAND = VAR >= 2;
    extern __shared__ __align__(16) u32 sm32[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const int kk = k + 1;
    const uint64_t base = high_tile_base<L>(blockIdx.x, kk);
    u32 v[kE];
    FirstAcc acc;
    if constexpr (MODE == FIRST_CHECK) {  // another tile failed: this one stores nothing either (in flight with the loads)
        if constexpr (VAR == 0) acc.hi[0] = *reinterpret_cast<volatile unsigned*>(abort);
        else asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(acc.hi[0]) : "l"(abort));
        if constexpr (VAR == 4) {  // ... and does not even load: a refused signal costs a few tiles, not a read pass
            if (__syncthreads_or(acc.hi[0] != 0u)) return;
        }
    }
    const unsigned long long* p = src + first_base(base) + first_off<L>(thread_part<C, 0>(lane, warp), k);
    if constexpr (LAND) {
        const uint32_t land = (uint32_t)__cvta_generic_to_shared(sm32) + threadIdx.x * 16u;
#pragma unroll
        for (int q = 0; q < 16; ++q)
            asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(land + q * (kNT * 16u)),
                         "l"(p + first_off<L>(reg_part<C, 0>(32 + 2 * q), k))
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        ulonglong2 t[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) t[q] = ld2x64(p + first_off<L>(reg_part<C, 0>(2 * q), k));
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            v[2 * q] = (u32)t[q].x;
            v[2 * q + 1] = (u32)t[q].y;
            first_test<MODE, CHK>(t[q], q, lim, acc);
        }
        // this thread's own copies: no CTA barrier needed to read them.  The warp barrier keeps ptxas from
        // hoisting the wait above the plain loads (which would then start a second round trip)
        __syncwarp();
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            ulonglong2 u;
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(u.x), "=l"(u.y) : "r"(land + q * (kNT * 16u)));
            v[32 + 2 * q] = (u32)u.x;
            v[32 + 2 * q + 1] = (u32)u.y;
            first_test<MODE, CHK>(u, q, lim, acc);
        }
    } else {
#pragma unroll
        for (int g = 0; g < kE; g += 16) {
            ulonglong2 t[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) t[q] = ld2x64(p + first_off<L>(reg_part<C, 0>(g + 2 * q), k));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                v[g + 2 * q] = (u32)t[q].x;
                v[g + 2 * q + 1] = (u32)t[q].y;
                first_test<MODE, CHK>(t[q], q, lim, acc);
            }
        }
    }
    BW_STRESS(67);
    high_rounds_store<L, MODE == FIRST_CHECK, LAND>(v, sm32, dst, base, kk, lane, warp,
                                                     MODE == FIRST_CHECK && first_bad<CHK>(acc, lim), tileflag, abort);
}

// The input test on the first 2^14 inputs only (one CTA): at n >= 33 a refused
// attempt costs two sweeps of 2^(n-14) returning CTAs, so signals whose first
// values already exceed lim (wide-valued data, config 5's sums) are turned
// away by this sample instead.
__global__ void __launch_bounds__(kNT) k32_sample(const unsigned long long* __restrict__ x, u32 lim, unsigned* abort) {
    u32 hi = 0, lo = 0;
    for (uint32_t j = threadIdx.x; j < (1u << kBits); j += kNT) {
        const unsigned long long y = x[j] + lim;
        hi |= (u32)(y >> 32);
        lo = max(lo, (u32)y);
    }
    if (hi != 0u || lo > 2u * lim) atomicExch(abort, 1u);
}

// Undo k32_first on the tiles it wrote (tileflag set): the int32 copy, the
// same r stages again (H H = 2^r I), >> r, stored as natural int64 over the
// bytes the tile read in the first place.
template <int L>
__global__ void __launch_bounds__(kNT, 2)
    k32_restore(const u32* __restrict__ src, unsigned long long* __restrict__ dst, int k, const unsigned* tileflag) {
    using C = CfgHighW<L>;
    static_assert(vec<C, 0>() == 2 && vec<C, 1>() == 4, "int32 pairs in, int64 pairs out");
    extern __shared__ __align__(16) u32 sm32[];
    if (*reinterpret_cast<const volatile unsigned*>(tileflag + blockIdx.x) == 0u) return;  // uniform per CTA
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const int kk = k + 1;
    const uint64_t base = high_tile_base<L>(blockIdx.x, kk);
    u32 v[kE];
    {
        const u32* p = src + base + high_off<L>(thread_part<C, 0>(lane, warp), kk);
#pragma unroll
        for (int j = 0; j < kE; j += 2) {
            const uint2 t = ld2(p + high_off<L>(reg_part<C, 0>(j), kk));
            v[j] = t.x;
            v[j + 1] = t.y;
        }
    }
    stages32<C, 0>(v);
    smem_store32<C, 0>(v, sm32, thread_part<C, 0>(lane, warp));
    __syncthreads();  // every load of the tile precedes every store over it
    const uint32_t tp = thread_part<C, 1>(lane, warp);
    smem_load32<C, 1>(v, sm32, tp);
    stages32<C, 1>(v);
    constexpr int r = kBits - L;
    unsigned long long* p = dst + first_base(base) + first_off<L>(tp, k);
#pragma unroll
    for (int j = 0; j < kE; j += 2) {
        ulonglong2 t;
        t.x = (unsigned long long)(long long)((int)v[j] >> r);
        t.y = (unsigned long long)(long long)((int)v[j + 1] >> r);
        *reinterpret_cast<ulonglong2*>(p + first_off<L>(reg_part<C, 1>(j), k)) = t;
    }
}
// int32 -> int64 low pass over stages 0..13 of every block.  src: the int32
// view offset by the read half (block b's copy at src + (b << 15)); dst: the
// int64 signal (block b at dst + (b << 14)).
// EX: the threshold extraction of the last pass (noisy.py:185-222 with
// |W| >= tau, as k_pass's): each sub-round's final values are tested in
// registers after their store; a warp holding a hit re-reads its stored
// values and appends (index, value) to the unordered hit list.
__device__ __noinline__ void low_extract_slow(const unsigned long long* o, uint64_t gbase, uint32_t tp, ExtractArgs ex) {
    using C = CfgLowW;
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {
        const uint32_t off = tp | reg_part<C, 2>(j);
        const u64 x = o[off];
        const bool h = hit_ge_u(x, ex.tau);
        const unsigned b = __ballot_sync(0xffffffffu, h);
        if (b) {
            const int leader = __ffs(b) - 1;
            unsigned long long first = 0;
            if ((int)lane == leader) first = atomicAdd(ex.count, (unsigned long long)__popc(b));
            first = __shfl_sync(0xffffffffu, first, leader);
            if (h) {
                const unsigned long long pos = first + __popc(b & ((1u << lane) - 1u));
                if (pos < ex.cap) {
                    ex.idx[pos] = (long long)(ex.base + gbase + off);
                    ex.val[pos] = (long long)x;
                }
            }
        }
    }
}

template <bool EX = false>
__global__ void __launch_bounds__(kNT, 2)
    k32_low(const u32* __restrict__ src, unsigned long long* __restrict__ dst, ExtractArgs ex) {
    using C = CfgLowW;
    extern __shared__ __align__(16) u32 sm32[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint64_t b = blockIdx.x;
    u32 v[kE];
    {
        const uint32_t tp = thread_part<C, 0>(lane, warp);
        const u32* p = src + (b << (kBits + 1)) + C::src_off(tp);
        static_assert(vec<C, 0>() == 4, "16-byte loads");
#pragma unroll
        for (int j = 0; j < kE; j += 4) {
            const uint4 t = ld4(p + C::src_off(reg_part<C, 0>(j)));
            v[j] = t.x;
            v[j + 1] = t.y;
            v[j + 2] = t.z;
            v[j + 3] = t.w;
        }
    }
    stages32<C, 0>(v);
    BW_STRESS(62);
    smem_store32<C, 0>(v, sm32, thread_part<C, 0>(lane, warp));
    BW_STRESS(63);
    __syncthreads();
    const uint32_t tp1 = thread_part<C, 1>(lane, warp);
    smem_load32<C, 1>(v, sm32, tp1);
    stages32<C, 1>(v);
    BW_STRESS(64);
    __syncthreads();  // every round-1 read is done before the slots are rewritten
    smem_store32<C, 1>(v, sm32, tp1);
    BW_STRESS(65);
    __syncthreads();
    unsigned long long* o = dst + (b << kBits);
    static_assert(vec<C, 2>() == 2, "int32 pairs from shared memory, int64 pairs to global");
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const uint32_t tp = thread_part<C, 2>(lane, warp) | ((uint32_t)s << C::SUB);
        const uint32_t st = C::slot(tp);
        unsigned long long w[32];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const uint2 t = *reinterpret_cast<const uint2*>(sm32 + (st ^ C::slot(reg_part<C, 2>(j))));
            w[j] = (unsigned long long)(long long)(int)t.x;
            w[j + 1] = (unsigned long long)(long long)(int)t.y;
        }
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if ((C::stage(2) >> C::reg(2, i)) & 1u) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (!((j >> i) & 1)) {
                        const unsigned long long a = w[j], c = w[j | (1 << i)];
                        w[j] = a + c;
                        w[j | (1 << i)] = a - c;
                    }
                }
            }
        }
        BW_STRESS(66);
        unsigned long long* p = o + tp;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            ulonglong2 t;
            t.x = w[j];
            t.y = w[j + 1];
            st_pass(reinterpret_cast<ulonglong2*>(p + reg_part<C, 2>(j)), t);
        }
        if constexpr (EX) {
            if (__any_sync(0xffffffffu, maybe_hit<32>(w, ex.tau)) && __any_sync(0xffffffffu, any_hit<32>(w, ex.tau)))
                low_extract_slow(o, b << kBits, tp, ex);
        }
    }
}
#endif  // __CUDACC__

}  // namespace w32
}  // namespace bw
