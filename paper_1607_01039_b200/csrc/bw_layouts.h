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
// Every CTA holds 2^13 elements of the tile (256 threads x 32 int64 in
// registers, two CTAs per SM).  Tiles of 2^14 / 2^15 elements are split over
// a thread-block cluster of 2 / 4 CTAs: the top q tile bits are the CTA's
// cluster rank ("pre" space).  Once every CTA-local stage is done, one
// transpose runs through distributed shared memory and swaps those rank bits
// with q already-staged local bits ("post" space), after which the former
// rank bits are local and get their stages.
//
// Inside a CTA every tile bit of the current space lives in one of three
// places: a register bit (5), a lane bit (5) or a warp bit (3).  A round is
// one such assignment; butterflies run only on register bits, and
// consecutive rounds are joined by a transpose through shared memory (slot of
// local index e is e + (e >> 5): every 8-byte access of every round is
// conflict-free per half-warp, which bw_plan_check verifies).  The same
// tables drive the device kernels, the host plan checker and the host
// emulator, so those check the addresses the kernels really touch.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define BW_HD __host__ __device__
#else
#define BW_HD
#endif

#ifndef BW_T13_MINB
#define BW_T13_MINB 2  // CTAs per SM the kernels are register-budgeted for
#endif

namespace bw {

constexpr int kCtaBits = 13;        // elements per CTA = 2^13 (64 KiB)
constexpr int kMaxHighBits = 10;    // stages per strided high-bits pass
constexpr int kRegOnlyMaxBits = 5;  // high passes this narrow need no smem
constexpr int kMaxClusterLog2 = 2;  // clusters of up to 4 CTAs

// Layout tables are packed 4 bits per entry (entry i = nibble i) so that the
// same constexpr functions fold to immediates in device code and run
// unchanged in the host checker / emulator.
BW_HD constexpr int nib(uint64_t packed, int i) { return (int)((packed >> (4 * i)) & 15u); }

// Common fields: T (tile bits), Q (log2 cluster size), R/W (register/warp
// bits), NR (rounds), XR (first round in post space; NR if no exchange),
// P(i) (local positions that take the rank bits after the exchange),
// MINB (CTAs per SM the register budget targets).  reg/lane/warp tables are
// VIRTUAL tile bits; stage(rd) is a mask of virtual tile bits.

// Fused low-bits pass over stages 0..12 (single CTA).
//   round 0: reg {0,9,10,11,12}  lane {1,2,3,5,4}  warp {6,7,8}
//   round 1: reg {1,2,3,4,5}     lane {0,6,7,8,9}  warp {10,11,12}
//   round 2: reg {0,6,7,8,12}    lane {1,2,3,5,4}  warp {9,10,11}
struct CfgLow13 {
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 3, XR = 3, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA90ull : rd == 1 ? 0x54321ull : 0xC8760ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 1 ? 0x98760ull : 0x45321ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x876ull : rd == 1 ? 0xCBAull : 0xBA9ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1E01u : rd == 1 ? 0x003Eu : 0x01C0u; }
    BW_HD static constexpr int P(int) { return 0; }
};

// Low-bits pass over stages 0..13: cluster of 2.  Round 0 stages the bits
// it holds in registers, then the rank bit (tile bit 13) swaps with tile
// bit 12 in the first transpose, which runs through DSMEM.  Lanes sit on
// tile bits 0..4 whenever a round writes remote memory, so every DSMEM store
// instruction covers 256 contiguous bytes.
//   round 0: reg {8..12}            lane {0,1,2,3,4}  warp {5,6,7}
//   round 1 (post): reg {0..4}      lane {5,6,7,8,9}  warp {10,11,13}
//   round 2 (post): reg {5,6,7,8,13} lane {0,1,2,3,4} warp {9,10,11}
struct CfgLow14c {
    static constexpr int T = 14, Q = 1, R = 5, W = 3, NR = 3, XR = 1, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA98ull : rd == 1 ? 0x43210ull : 0xD8765ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 1 ? 0x98765ull : 0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x765ull : rd == 1 ? 0xDBAull : 0xBA9ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1F00u : rd == 1 ? 0x001Fu : 0x20E0u; }
    BW_HD static constexpr int P(int) { return 12; }
};

// The same layout budgeted for three CTAs per SM (register cap 80; the
// BW_LOW14_MINB3=1 experiment of the n = 34 low pass: 57.4 ms = 4.79 TB/s
// against 46.4 ms with two, profiles/r02_evidence/low14_minb3_negative.log).
struct CfgLow14c3 : CfgLow14c {
    static constexpr int MINB = 3;
};

// Low-bits pass over stages 0..14: cluster of 4; the rank bits (13, 14)
// swap with tile bits 11, 12 in the first (DSMEM) transpose.
//   round 0: reg {8..12}              lane {0,1,2,3,4}  warp {5,6,7}
//   round 1 (post): reg {0..4}        lane {5,6,7,8,9}  warp {10,13,14}
//   round 2 (post): reg {5,6,7,13,14} lane {0,1,2,3,4}  warp {8,9,10}
struct CfgLow15c {
    static constexpr int T = 15, Q = 2, R = 5, W = 3, NR = 3, XR = 1, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA98ull : rd == 1 ? 0x43210ull : 0xED765ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 1 ? 0x98765ull : 0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x765ull : rd == 1 ? 0xEDAull : 0xA98ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1F00u : rd == 1 ? 0x001Fu : 0x60E0u; }
    BW_HD static constexpr int P(int i) { return 11 + i; }
};

// Strided high-bits pass with 6..8 stage rows (tile bits L..12, L = 13 - r).
//   round 0: reg {8..12}  lane {0,1,2,3,4}  warp {5,6,7}
//   round 1: reg {3..7}   lane {0,1,2,8,9}  warp {10,11,12}
struct CfgHigh13 {
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 2, XR = 2, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA98ull : 0x76543ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 0 ? 0x43210ull : 0x98210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x765ull : 0xCBAull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1F00u : 0x00F8u; }
    BW_HD static constexpr int P(int) { return 0; }
};

// High-bits pass over rows L..13 (r = 14 - L: 9 at L = 5, 10 at L = 4):
// cluster of 2.  The rank bit (tile bit 13, the top row) swaps with tile
// bit 12 in the only transpose, which runs through DSMEM.
//   round 0: reg {8..12}          lane {0,1,2,3,4}  warp {5,6,7}
//   round 1 (post): reg {4,5,6,7,13}  lane {0,1,2,3,8}  warp {9,10,11}
struct CfgHigh14c {
    static constexpr int T = 14, Q = 1, R = 5, W = 3, NR = 2, XR = 1, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA98ull : 0xD7654ull, i); }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 0 ? 0x43210ull : 0x83210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x765ull : 0xBA9ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1F00u : 0x20F0u; }
    BW_HD static constexpr int P(int) { return 12; }
};

// High-bits pass over rows L..14 (r = 15 - L: 10 at L = 5): cluster of 4.
// The rank bits (13, 14) swap with tile bits 11, 12 in the DSMEM transpose.
//   round 0: reg {8..12}           lane {0,1,2,3,4}  warp {5,6,7}
//   round 1 (post): reg {5,6,7,13,14}  lane {0,1,2,3,4}  warp {8,9,10}
struct CfgHigh15c {
    static constexpr int T = 15, Q = 2, R = 5, W = 3, NR = 2, XR = 1, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) { return nib(rd == 0 ? 0xCBA98ull : 0xED765ull, i); }
    BW_HD static constexpr int lane(int, int i) { return nib(0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) { return nib(rd == 0 ? 0x765ull : 0xA98ull, i); }
    BW_HD static constexpr uint32_t stage(int rd) { return rd == 0 ? 0x1F00u : 0x60E0u; }
    BW_HD static constexpr int P(int i) { return 11 + i; }
};

// Split-row variants of the 1- and 2-CTA high passes: the same rounds, but
// the tile's rows are two runs of global bits (see split_rows below).
struct CfgHigh13S : CfgHigh13 {
    static constexpr bool SPLIT = true;
};
struct CfgHigh14cS : CfgHigh14c {
    static constexpr bool SPLIT = true;
};

// Strided high-bits pass with <= 5 stage rows: register-only, no shared
// memory; tile bits 8..12 in registers.
//   round 0: reg {8..12}  lane {0..4}  warp {5,6,7}
struct CfgReg {
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 1, XR = 1, MINB = 1, PAD = 1;
    BW_HD static constexpr int reg(int, int i) { return nib(0xCBA98ull, i); }
    BW_HD static constexpr int lane(int, int i) { return nib(0x43210ull, i); }
    BW_HD static constexpr int warp(int, int i) { return nib(0x765ull, i); }
    BW_HD static constexpr uint32_t stage(int) { return 0x1F00u; }
    BW_HD static constexpr int P(int) { return 0; }
};

// ---- float64 layouts ---------------------------------------------------
// numpy's float64 result depends on the order of the stages (rounding), so
// the float64 passes apply every element's stages in ascending bit order:
// rounds take increasing stage bits and each round's register indices list
// them in increasing order (bw_plan_check_f64 verifies this).
//
// Fused low-bits pass over stages 0..12, four rounds (round 0 only loads):
//   round 0: reg {8..12}          lane {0..4}  warp {5,6,7}
//   round 1: reg {0..4}           lane {5..9}  warp {10,11,12}  stages 0..4
//   round 2: reg {5..9}           lane {0..4}  warp {10,11,12}  stages 5..9
//   round 3: reg {10,11,12,5,6}   lane {0..4}  warp {7,8,9}     stages 10..12
struct CfgLow13F {
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 4, XR = 4, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(rd == 0 ? 0xCBA98ull : rd == 1 ? 0x43210ull : rd == 2 ? 0x98765ull : 0x65CBAull, i);
    }
    BW_HD static constexpr int lane(int rd, int i) { return nib(rd == 1 ? 0x98765ull : 0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) {
        return nib(rd == 0 ? 0x765ull : rd == 3 ? 0x987ull : 0xCBAull, i);
    }
    BW_HD static constexpr uint32_t stage(int rd) {
        return rd == 0 ? 0u : rd == 1 ? 0x001Fu : rd == 2 ? 0x03E0u : 0x1C00u;
    }
    BW_HD static constexpr int P(int) { return 0; }
};

// The same four rounds with 16-byte global accesses: round 0 holds tile
// bit 0 in a register (element pairs) and stages only it, the last round
// holds it again for paired stores.
//   round 0: reg {0,9,10,11,12}  lane {1,2,3,5,4}  warp {6,7,8}    stage 0
//   round 1: reg {1..5}          lane {0,6,7,8,9}  warp {10,11,12} stages 1..5
//   round 2: reg {6..10}         lane {0..4}       warp {5,11,12}  stages 6..10
//   round 3: reg {0,11,12,6,7}   lane {1,2,3,5,4}  warp {8,9,10}   stages 11,12
struct CfgLow13FV {
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 4, XR = 4, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(rd == 0 ? 0xCBA90ull : rd == 1 ? 0x54321ull : rd == 2 ? 0xA9876ull : 0x76CB0ull, i);
    }
    BW_HD static constexpr int lane(int rd, int i) {  // lanes {1,2,3,5,4}: conflict-free with the pad
        return nib(rd == 1 ? 0x98760ull : rd == 2 ? 0x43210ull : 0x45321ull, i);
    }
    BW_HD static constexpr int warp(int rd, int i) {
        return nib(rd == 0 ? 0x876ull : rd == 1 ? 0xCBAull : rd == 2 ? 0xCB5ull : 0xA98ull, i);
    }
    BW_HD static constexpr uint32_t stage(int rd) {
        return rd == 0 ? 0x0001u : rd == 1 ? 0x003Eu : rd == 2 ? 0x07C0u : 0x1800u;
    }
    BW_HD static constexpr int P(int) { return 0; }
};

// Strided high-bits pass with LL column bits (r = 13 - LL = 6..8 rows,
// tile bits LL..12), ascending: round 0 stages the five lowest rows, round 1
// the rest; lanes stay on columns 0..4 (256-byte accesses).
//   LL=5: round 0 reg {5..9}  warp {10,11,12}; round 1 reg {10,11,12,5,6} warp {7,8,9}
//   LL=6: round 0 reg {6..10} warp {5,11,12};  round 1 reg {11,12,5,6,7}  warp {8,9,10}
//   LL=7: round 0 reg {7..11} warp {5,6,12};   round 1 reg {12,5,6,7,8}   warp {9,10,11}
template <int LL>
struct CfgHigh13F {
    static_assert(LL >= 5 && LL <= 7, "float64 high pass covers 6..8 rows");
    static constexpr int T = 13, Q = 0, R = 5, W = 3, NR = 2, XR = 2, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(LL == 5 ? (rd == 0 ? 0x98765ull : 0x65CBAull)
                   : LL == 6 ? (rd == 0 ? 0xA9876ull : 0x765CBull)
                             : (rd == 0 ? 0xBA987ull : 0x8765Cull),
                   i);
    }
    BW_HD static constexpr int lane(int, int i) { return nib(0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) {
        return nib(LL == 5 ? (rd == 0 ? 0xCBAull : 0x987ull)
                   : LL == 6 ? (rd == 0 ? 0xCB5ull : 0xA98ull)
                             : (rd == 0 ? 0xC65ull : 0xBA9ull),
                   i);
    }
    BW_HD static constexpr uint32_t stage(int rd) {
        return rd == 0 ? (0x1Fu << LL) : (0x1FFFu << (LL + 5)) & 0x1FFFu;
    }
    BW_HD static constexpr int P(int) { return 0; }
};

// Strided high-bits pass over rows LL..13 (r = 14 - LL = 9 / 10) on a
// cluster of 2, ascending: round 0 stages the five lowest rows, the DSMEM
// transpose brings the rank row (tile bit 13) into the CTA at local
// position P = LL + 4 (already staged), round 1 stages the rest in order.
//   LL=5: round 0 reg {5..9}  lane {0..4}        warp {10,11,12}  P = 9
//         round 1 reg {10,11,12,13,5}  lane {0..4}  warp {6,7,8}
//   LL=4: round 0 reg {4..8}  lane {0,1,2,3,12}  warp {9,10,11}   P = 8
//         round 1 reg {9..13}  lane {0..4}          warp {5,6,7}
template <int LL>
struct CfgHigh14cF {
    static_assert(LL == 4 || LL == 5, "float64 cluster pass covers 9 or 10 rows");
    static constexpr int T = 14, Q = 1, R = 5, W = 3, NR = 2, XR = 1, MINB = BW_T13_MINB, PAD = 1;
    BW_HD static constexpr int reg(int rd, int i) {
        return nib(LL == 5 ? (rd == 0 ? 0x98765ull : 0x5DCBAull) : (rd == 0 ? 0x87654ull : 0xDCBA9ull), i);
    }
    BW_HD static constexpr int lane(int rd, int i) { return nib(LL == 4 && rd == 0 ? 0xC3210ull : 0x43210ull, i); }
    BW_HD static constexpr int warp(int rd, int i) {
        return nib(LL == 5 ? (rd == 0 ? 0xCBAull : 0x876ull) : (rd == 0 ? 0xBA9ull : 0x765ull), i);
    }
    BW_HD static constexpr uint32_t stage(int rd) {
        return rd == 0 ? (0x1Fu << LL) : (0x3FFFu << (LL + 5)) & 0x3FFFu;
    }
    BW_HD static constexpr int P(int) { return LL + 4; }
};

template <class C>
struct Dims {
    static constexpr int E = 1 << C::R;               // elements per thread
    static constexpr int NT = 32 << C::W;             // threads per CTA
    static constexpr int CTA = 1 << kCtaBits;         // elements per CTA
    static constexpr int SMEM_ELEMS = C::NR > 1 ? CTA + C::PAD * (CTA >> 5) : 0;
    static constexpr int CLUSTER = 1 << C::Q;
    // dynamic shared memory: the transpose buffer, plus one mbarrier for the
    // DSMEM exchange of cluster configs
    static constexpr int SMEM_BYTES = SMEM_ELEMS * 8 + (C::Q > 0 ? 8 : 0);
};

// Padded shared-memory slot of local index e; additive over disjoint bit sets.
BW_HD constexpr uint32_t smem_slot(uint32_t e) { return e + (e >> 5); }
template <class C>
BW_HD constexpr uint32_t smem_slot_c(uint32_t e) { return e + C::PAD * (e >> 5); }

// Round RD moves element pairs (tile bits 0) as 16-byte shared-memory words
// (configs with PAD = 2 keep pairs 16-byte aligned; a vectorised 2-CTA low
// pass built on it measured 5.75 vs 5.92 TB/s and was dropped).
template <class C, int RD>
BW_HD constexpr bool vec_smem() { return C::PAD == 2 && C::reg(RD, 0) == 0; }

// Tile index (virtual bits) contributed by register index j in round RD.
template <class C, int RD>
BW_HD constexpr uint32_t reg_part(int j) {
    uint32_t e = 0;
    for (int i = 0; i < C::R; ++i)
        if ((j >> i) & 1) e |= 1u << C::reg(RD, i);
    return e;
}

// Tile index (virtual bits) contributed by (lane, warp) in round RD.
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

// Mask of the tile bits held by lanes and warps in round RD.
template <class C, int RD>
BW_HD constexpr uint32_t thread_part_bits() {
    uint32_t m = 0;
    for (int i = 0; i < 5; ++i) m |= 1u << C::lane(RD, i);
    for (int i = 0; i < C::W; ++i) m |= 1u << C::warp(RD, i);
    return m;
}

// Mask of the positions P(0..Q-1) (post-space rank bits).
template <class C>
BW_HD constexpr uint32_t p_mask() {
    uint32_t m = 0;
    for (int i = 0; i < C::Q; ++i) m |= 1u << C::P(i);
    return m;
}

// Local (per-CTA) index of virtual index v in round RD's space.  Pre space:
// identity on bits 0..12.  Post space: virtual bit 13+i sits at local P(i).
// Linear over disjoint bit sets (bits are moved, never combined).
template <class C, int RD>
BW_HD constexpr uint32_t to_local(uint32_t v) {
    if (RD < C::XR || C::Q == 0) return v;
    uint32_t e = v & ((1u << kCtaBits) - 1u);
    for (int i = 0; i < C::Q; ++i) e |= ((v >> (kCtaBits + i)) & 1u) << C::P(i);
    return e;
}

// Virtual bits fixed by the CTA's cluster rank in round RD's space.
template <class C, int RD>
BW_HD constexpr uint32_t rank_bits(uint32_t rank) {
    if (C::Q == 0) return 0;
    if (RD < C::XR) return rank << kCtaBits;
    uint32_t v = 0;
    for (int i = 0; i < C::Q; ++i) v |= ((rank >> i) & 1u) << C::P(i);
    return v;
}

// Stage mask of round RD for a tile whose low L bits are columns.
template <class C, int RD, int L>
BW_HD constexpr uint32_t stage_mask() {
    return L >= C::T ? C::stage(RD) : (C::stage(RD) & ~((1u << L) - 1u));
}

// ---- split rows ----------------------------------------------------------
// A high pass normally stages one run of global bits [k, k+r).  A SPLIT pass
// stages two runs: tile row i (0 <= i < r) is global bit k + i for i < a and
// k2 + (i - a) for i >= a (k + a <= k2).  Its kernels receive the three
// numbers packed in their int k argument.  Split rows let a plan give a
// pass the low rows {k..k+a-1} of a large-stride pass: the tile then spans
// 2^(r-a) DRAM pages instead of 2^r (n = 34: rows {14..17} u {28..33} run at
// 6.27 TB/s, rows {24..33} at 5.77 -- tools/mb_split.cu).  Stages on
// distinct bits commute in Z/2^64, so any such plan is bit-identical for
// int64 (float64 keeps its ascending one-run plans).
BW_HD constexpr int split_pack(int k, int a, int k2) { return k | (a << 8) | (k2 << 16); }
BW_HD constexpr int split_k(int packed) { return packed & 255; }
BW_HD constexpr int split_a(int packed) { return (packed >> 8) & 255; }
BW_HD constexpr int split_k2(int packed) { return packed >> 16; }

// C::SPLIT if the config declares it, else false.
template <class C, class = void>
struct SplitOf {
    static constexpr bool value = false;
};
template <class C>
struct SplitOf<C, decltype(void(C::SPLIT))> {
    static constexpr bool value = C::SPLIT;
};

// Global element offset (relative to the tile base) of tile index e.
// Linear over disjoint bit sets (every tile bit maps to one global bit).
template <int T, int L, bool S = false>
BW_HD inline uint64_t global_off(uint32_t e, int k) {
    if (L >= T) return e;
    const uint64_t col = e & ((1u << L) - 1u);
    const uint32_t row = e >> L;
    if constexpr (!S) {
        return col + ((uint64_t)row << k);
    } else {
        const int a = split_a(k);
        return col + ((uint64_t)(row & ((1u << a) - 1u)) << split_k(k)) + ((uint64_t)(row >> a) << split_k2(k));
    }
}

// Global index of element 0 of tile `b` for a pass over bits [k, k+T-L)
// (split: the free global bits [L, k), [k+a, k2), [k2+r-a, ...) take the
// tile id's bits in ascending order, so neighbouring tiles are neighbouring
// column groups, as for one run).
template <int T, int L, bool S = false>
BW_HD inline uint64_t tile_base(uint64_t b, int k) {
    if (L >= T) return b << T;
    if constexpr (!S) {
        const int mid = k - L;  // global bits L..k-1 come from the low tile-id bits
        return ((b & ((1ull << mid) - 1ull)) << L) | ((b >> mid) << (k + T - L));
    } else {
        const int k1 = split_k(k), a = split_a(k), k2 = split_k2(k);
        const int m1 = k1 - L, m2 = k2 - (k1 + a);
        const uint64_t lo = b & ((1ull << m1) - 1ull);
        const uint64_t mid = (b >> m1) & ((1ull << m2) - 1ull);
        const uint64_t hi = b >> (m1 + m2);
        return (lo << L) | (mid << (k1 + a)) | (hi << (k2 + (T - L) - a));
    }
}

}  // namespace bw
