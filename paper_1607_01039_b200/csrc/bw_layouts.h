// bw_layouts.h -- tile layouts of the FWHT pass kernels (host + device).
//
// A pass transforms the signal tile by tile.  A tile is 2^T elements whose
// "tile bits" 0..T-1 map onto global index bits:
//     tile bit b <  L  ->  global bit b            (contiguous columns)
//     tile bit b >= L  ->  global bit k + (b - L)  (the pass's stage rows)
// For the low-bits pass L = T (the tile is 2^T contiguous elements, stages
// 0..T-1: external.py:238-254 `_initial_pass` with 2^B = the tile).  For a
// high-bits pass the tile is 2^(T-L) rows at stride 2^k times 2^L contiguous
// columns, and the pass applies stages k..k+T-L-1 (external.py:272-283
// `_blocked_stage_pass`, merging T-L stages per HBM round trip).
//
// Inside a CTA every tile bit lives in one of three places: a register bit
// (a thread holds 2^R elements), a lane bit (5) or a warp bit (W).  A round
// is one such assignment; butterflies run only on register bits, and
// consecutive rounds are joined by a transpose through shared memory
// (padded address e + (e >> 5), chosen so that every 8-byte access of every
// round is conflict free per half-warp -- see DESIGN.md).  The same tables
// drive the device kernels and the host plan checker (bw_plan_check), so the
// checker verifies the addresses the kernels really touch.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BW_HD __host__ __device__
#else
#define BW_HD
#endif

namespace bw {

constexpr int kLowBits = 14;      // stages fused into the low-bits pass
constexpr int kMaxHighBits = 10;  // stages per strided high-bits pass
constexpr int kRegOnlyMaxBits = 5;

// Layout tables are packed 4 bits per entry (entry i = nibble i) so that
// the same constexpr functions fold to immediates in device code and run
// unchanged in the host plan checker.
BW_HD constexpr int nib(uint64_t packed, int i) { return (int)((packed >> (4 * i)) & 15u); }

// Fused low-bits pass: 2^14 contiguous int64 (128 KiB) per CTA, 512 threads,
// 32 elements per thread; rounds stage {0,10..13}, {1..5}, {6..9}.
// Rounds 0 and 2 put tile bit 0 in register bit 0 -> 16-byte global accesses.
//   round 0: reg {0,10,11,12,13}  lane {1,2,3,5,4}  warp {6,7,8,9}
//   round 1: reg {1,2,3,4,5}      lane {0,6,7,8,9}  warp {10..13}
//   round 2: reg {0,6,7,8,9}      lane {1,2,3,5,4}  warp {10..13}
struct CfgLow {
    static constexpr int T = 14, R = 5, W = 4, NR = 3;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xDCBA0ull : rd == 1 ? 0x54321ull : 0x98760ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 1 ? 0x98760ull : 0x45321ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x9876ull : 0xDCBAull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x3C01u : rd == 1 ? 0x003Eu : 0x03C0u; }
};

// Strided high-bits pass with 6..10 stage rows: 2^14 elements per CTA,
// 512 threads; rounds stage tile bits {9..13} and {L..8}; one transpose.
//   round 0: reg {9..13}  lane {0,1,2,3,4}  warp {5,6,7,8}
//   round 1: reg {4..8}   lane {0,1,2,3,9}  warp {10..13}
struct CfgHigh {
    static constexpr int T = 14, R = 5, W = 4, NR = 2;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xDCBA9ull : 0x87654ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 0 ? 0x43210ull : 0x93210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x8765ull : 0xDCBAull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x3E00u : 0x01F0u; }
};

// Strided high-bits pass with <= 5 stage rows: register-only, no shared
// memory; 2^13-element tiles, 256 threads x 32 elements, tile bits 8..12 in
// registers (2 CTAs per SM).
//   round 0: reg {8..12}  lane {0..4}  warp {5,6,7}
struct CfgReg {
    static constexpr int T = 13, R = 5, W = 3, NR = 1;
    BW_HD static constexpr int reg(int, int i) { return nib(0xCBA98ull, i); }
    BW_HD static constexpr int lane(int, int i) { return nib(0x43210ull, i); }
    BW_HD static constexpr int warp(int, int i) { return nib(0x765ull, i); }
    BW_HD static constexpr uint32_t stage(int) { return 0x1F00u; }
};

template <class C>
struct Dims {
    static constexpr int E = 1 << C::R;              // elements per thread
    static constexpr int NT = 32 << C::W;            // threads per CTA
    static constexpr int TILE = 1 << C::T;           // elements per tile
    static constexpr int SMEM_ELEMS = C::NR > 1 ? TILE + (TILE >> 5) : 0;
};

// Padded shared-memory slot of tile index e; additive over disjoint bit sets.
BW_HD constexpr uint32_t smem_slot(uint32_t e) { return e + (e >> 5); }

// Tile index contributed by register index j in round RD.
template <class C, int RD>
BW_HD constexpr uint32_t reg_part(int j) {
    uint32_t e = 0;
    for (int i = 0; i < C::R; ++i)
        if ((j >> i) & 1) e |= 1u << C::reg(RD, i);
    return e;
}

// Tile index contributed by (lane, warp) in round RD.
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
    for (int i = 0; i < C::W; ++i) e |= ((warp >> i) & 1u) << C::warp(RD, i);
    return e;
}

// Stage mask of round RD for a tile whose low L bits are columns.
template <class C, int RD, int L>
BW_HD constexpr uint32_t stage_mask() {
    return L >= C::T ? C::stage(RD) : (C::stage(RD) & ~((1u << L) - 1u));
}

// Global element offset (relative to the tile base) of tile index e.
template <int T, int L>
BW_HD inline uint64_t global_off(uint32_t e, int k) {
    if (L >= T) return e;
    return (uint64_t)(e & ((1u << L) - 1u)) + ((uint64_t)(e >> L) << k);
}

// Global index of element 0 of tile `b` for a pass over bits [k, k+T-L).
template <int T, int L>
BW_HD inline uint64_t tile_base(uint64_t b, int k) {
    if (L >= T) return b << T;
    const int mid = k - L;  // global bits L..k-1 come from the low tile-id bits
    return ((b & ((1ull << mid) - 1ull)) << L) | ((b >> mid) << (k + T - L));
}

}  // namespace bw
