// bw_kernels.cuh -- sm_100a kernels of the B200 FWHT.
//
// All arithmetic is on uint64 bit patterns: two's-complement add/sub wraps
// modulo 2^64 exactly like numpy int64 (core.py:113-115), so every kernel is
// bit-identical to the reference for any input and any stage order.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "bw_layouts.h"

namespace bw {

typedef unsigned long long u64;

// Race stress (a build with -DBW_RACE_STRESS, tools/race_stress.sh): at every
// synchronisation point of the pass kernels, about one warp in four sleeps a
// pseudo-random 0..~2 us, so the orders in which CTAs and warps reach the
// cluster barriers, the DSMEM exchange, the mbarrier waits and the shared-
// memory transposes vary from run to run.  A missing or misplaced barrier
// then shows up as a result that differs from the oracle.  (The pool has
// compute-sanitizer closed; this is the dynamic check that replaces it.)
#ifdef BW_RACE_STRESS
__device__ __forceinline__ void race_stress(uint32_t id) {
    uint32_t h = blockIdx.x * 0x9E3779B1u ^ (threadIdx.x >> 5) * 0x85EBCA6Bu ^ id * 0xC2B2AE35u;
    h ^= (uint32_t)clock64() & 0xffu;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if ((h & 3u) == 0u) __nanosleep((h >> 16) & 2047u);
}
#define BW_STRESS(id) ::bw::race_stress(id)
#else
#define BW_STRESS(id) ((void)0)
#endif

// Cache policy of the pass kernels' global accesses (A/B knob: 0 = .cs
// streaming, 1 = .cg, 2 = default, 3 = default + L2::256B fetch size).
// Measured on B200 (profiles/r01_*): default loads lift the vectorised low
// pass from 6.4 to 7.0 TB/s; the 256-byte L2 fetch makes every DRAM access
// cover two neighbouring 128-byte row segments (the next tile's, already in
// L2 when that tile loads): 10-stage passes +1.5-2.2%, 5-stage register
// passes +5% (profiles/r01_shapes_l2_256B.json).  So: loads with L2::256B,
// plain stores.
#ifndef BW_LD_POLICY
#define BW_LD_POLICY 3
#endif
#ifndef BW_ST_POLICY
#define BW_ST_POLICY 2
#endif
template <class T>
__device__ __forceinline__ T ld_pass(const T* p) {
    if constexpr (BW_LD_POLICY == 0) return __ldcs(p);
    else if constexpr (BW_LD_POLICY == 1) return __ldcg(p);
    else if constexpr (BW_LD_POLICY == 3) {  // L2 fetch granularity 256 B (experiment)
        if constexpr (sizeof(T) == 16) {
            T v;
            asm volatile("ld.global.L2::256B.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
            return v;
        } else {
            T v;
            asm volatile("ld.global.L2::256B.u64 %0, [%1];" : "=l"(v) : "l"(p));
            return v;
        }
    } else return *p;
}
// Any 2- to 16-byte load with the passes' L2::256B fetch size (the mapped
// passes' narrow and pair types).
template <class T>
__device__ __forceinline__ T ld_any(const T* p) {
    T v;
    if constexpr (sizeof(T) == 16) {
        unsigned long long a, b;
        asm volatile("ld.global.L2::256B.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
        memcpy(&v, &a, 8);
        memcpy(reinterpret_cast<char*>(&v) + 8, &b, 8);
    } else if constexpr (sizeof(T) == 8) {
        unsigned long long a;
        asm volatile("ld.global.L2::256B.u64 %0, [%1];" : "=l"(a) : "l"(p));
        memcpy(&v, &a, 8);
    } else if constexpr (sizeof(T) == 4) {
        unsigned a;
        asm volatile("ld.global.L2::256B.u32 %0, [%1];" : "=r"(a) : "l"(p));
        memcpy(&v, &a, 4);
    } else {
        static_assert(sizeof(T) == 2, "2-16 byte loads");
        unsigned short a;
        asm volatile("ld.global.L2::256B.u16 %0, [%1];" : "=h"(a) : "l"(p));
        memcpy(&v, &a, 2);
    }
    return v;
}

template <class T>
__device__ __forceinline__ void st_pass(T* p, const T& v) {
    if constexpr (BW_ST_POLICY == 0) __stcs(p, v);
    else if constexpr (BW_ST_POLICY == 1) __stcg(p, v);
    else *p = v;
}

// ---------------------------------------------------------------------------
// Pass engine (kernels K1 low-bits, K2 high-bits, register-only high-bits).
// ---------------------------------------------------------------------------

// One butterfly on bit patterns: int64 (wrapping) or float64 (IEEE add /
// sub, single rounding each, exactly numpy's a + b and a - b).
template <bool FP>
__device__ __forceinline__ void butterfly(u64& x, u64& y) {
    if constexpr (FP) {
        const double a = __longlong_as_double((long long)x), b = __longlong_as_double((long long)y);
        x = (u64)__double_as_longlong(__dadd_rn(a, b));
        y = (u64)__double_as_longlong(__dsub_rn(a, b));
    } else {
        const u64 a = x, b = y;
        x = a + b;
        y = a - b;
    }
}

// Stages of round RD, register index i = 0..R-1 in order (for float64
// configs that order is ascending in the stage bit).
template <class C, int RD, int L, bool FP = false>
__device__ __forceinline__ void apply_stages(u64 (&v)[Dims<C>::E]) {
    constexpr int E = Dims<C>::E;
    constexpr uint32_t mask = stage_mask<C, RD, L>();
#pragma unroll
    for (int i = 0; i < C::R; ++i) {
        if ((mask >> C::reg(RD, i)) & 1u) {
#pragma unroll
            for (int j = 0; j < E; ++j) {
                if (!((j >> i) & 1)) butterfly<FP>(v[j], v[j | (1 << i)]);
            }
        }
    }
}

// Round RD has tile bit 0 as register bit 0: global access as 16-byte pairs.
template <class C, int RD, int L>
struct VecAccess {
    static constexpr bool value = (C::reg(RD, 0) == 0) && (L >= 1);
};

template <class C, int RD, int T, int L>
__device__ __forceinline__ void load_global(u64 (&v)[Dims<C>::E], const u64* __restrict__ g,
                                           uint32_t tp, int k) {
    constexpr int E = Dims<C>::E;
    const u64* p = g + global_off<T, L, SplitOf<C>::value>(tp, k);
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const uint64_t off = global_off<T, L, SplitOf<C>::value>(reg_part<C, RD>(j), k);
        if constexpr (VecAccess<C, RD, L>::value) {
            if ((j & 1) == 0) {
                const ulonglong2 t = ld_pass(reinterpret_cast<const ulonglong2*>(p + off));
                v[j] = t.x;
                v[j + 1] = t.y;
            }
        } else {
            v[j] = ld_pass(p + off);
        }
    }
}

// Widening load (int32 / int16 / int8 source, int64 registers) for the
// out-of-place first pass of bw_fwht_widen_i32 and of the narrow-wire
// multi-device transform: same addressing, SB-byte elements.
template <int SB>
struct NarrowType;
template <>
struct NarrowType<4> {
    typedef int one;
    typedef int2 pair;
};
template <>
struct NarrowType<2> {
    typedef short one;
    typedef short2 pair;
};
template <>
struct NarrowType<1> {
    typedef signed char one;
    typedef char2 pair;
};

template <class C, int RD, int T, int L, int SB>
__device__ __forceinline__ void load_global_narrow(u64 (&v)[Dims<C>::E], const void* __restrict__ src, uint32_t tp,
                                                   int k) {
    typedef typename NarrowType<SB>::one S1;
    typedef typename NarrowType<SB>::pair S2;
    constexpr int E = Dims<C>::E;
    const S1* p = reinterpret_cast<const S1*>(src) + global_off<T, L, SplitOf<C>::value>(tp, k);
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const uint64_t off = global_off<T, L, SplitOf<C>::value>(reg_part<C, RD>(j), k);
        if constexpr (VecAccess<C, RD, L>::value) {
            if ((j & 1) == 0) {
                const S2 t = __ldcs(reinterpret_cast<const S2*>(p + off));
                v[j] = (u64)(long long)(S1)t.x;
                v[j + 1] = (u64)(long long)(S1)t.y;
            }
        } else {
            v[j] = (u64)(long long)__ldcs(p + off);
        }
    }
}

template <class C, int RD, int T, int L>
__device__ __forceinline__ void store_global(const u64 (&v)[Dims<C>::E], u64* __restrict__ g,
                                             uint32_t tp, int k) {
    constexpr int E = Dims<C>::E;
    u64* p = g + global_off<T, L, SplitOf<C>::value>(tp, k);
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const uint64_t off = global_off<T, L, SplitOf<C>::value>(reg_part<C, RD>(j), k);
        if constexpr (VecAccess<C, RD, L>::value) {
            if ((j & 1) == 0) {
                ulonglong2 t;
                t.x = v[j];
                t.y = v[j + 1];
                st_pass(reinterpret_cast<ulonglong2*>(p + off), t);
            }
        } else {
            st_pass(p + off, v[j]);
        }
    }
}

// Split-row passes: the element offset of every register index of the load
// round and of the store round, computed once on the host (bw_abi
// split_table) and read straight from the kernel's parameter space -- one
// 64-bit add per element, where evaluating the two-run row map per element
// measured 40% more instructions and 5.2 instead of ~6.2 TB/s.
struct SplitTab {
    unsigned long long ld[32];
    unsigned long long st[32];
};

template <class C, int T, int L>
__device__ __forceinline__ void load_global_tab(u64 (&v)[Dims<C>::E], const u64* __restrict__ g, uint32_t tp,
                                                int k, const SplitTab& tab) {
    static_assert(Dims<C>::E == 32 && !VecAccess<C, 0, L>::value, "split passes use 8-byte accesses");
    const u64* p = g + global_off<T, L, true>(tp, k);
#pragma unroll
    for (int j = 0; j < Dims<C>::E; ++j) v[j] = ld_pass(p + tab.ld[j]);
}

template <class C, int T, int L>
__device__ __forceinline__ void store_global_tab(const u64 (&v)[Dims<C>::E], u64* __restrict__ g, uint32_t tp,
                                                 int k, const SplitTab& tab) {
    static_assert(Dims<C>::E == 32 && !VecAccess<C, C::NR - 1, L>::value, "split passes use 8-byte accesses");
    u64* p = g + global_off<T, L, true>(tp, k);
#pragma unroll
    for (int j = 0; j < Dims<C>::E; ++j) st_pass(p + tab.st[j], v[j]);
}

template <class C, int RD>
__device__ __forceinline__ void store_smem(const u64 (&v)[Dims<C>::E], u64* sm, uint32_t tp) {
    u64* p = sm + smem_slot_c<C>(to_local<C, RD>(tp));
#pragma unroll
    for (int j = 0; j < Dims<C>::E; ++j) {
        if constexpr (vec_smem<C, RD>()) {
            if ((j & 1) == 0) {
                ulonglong2 t;
                t.x = v[j];
                t.y = v[j + 1];
                *reinterpret_cast<ulonglong2*>(p + smem_slot_c<C>(to_local<C, RD>(reg_part<C, RD>(j)))) = t;
            }
        } else {
            p[smem_slot_c<C>(to_local<C, RD>(reg_part<C, RD>(j)))] = v[j];
        }
    }
}

template <class C, int RD>
__device__ __forceinline__ void load_smem(u64 (&v)[Dims<C>::E], const u64* sm, uint32_t tp) {
    const u64* p = sm + smem_slot_c<C>(to_local<C, RD>(tp));
#pragma unroll
    for (int j = 0; j < Dims<C>::E; ++j) {
        if constexpr (vec_smem<C, RD>()) {
            if ((j & 1) == 0) {
                const ulonglong2 t =
                    *reinterpret_cast<const ulonglong2*>(p + smem_slot_c<C>(to_local<C, RD>(reg_part<C, RD>(j))));
                v[j] = t.x;
                v[j + 1] = t.y;
            }
        } else {
            v[j] = p[smem_slot_c<C>(to_local<C, RD>(reg_part<C, RD>(j)))];
        }
    }
}

// ---- thread-block-cluster plumbing (DSMEM) ---------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, u64 v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
// Remote store that also signals `bytes` of transaction completion on the
// destination CTA's mbarrier (no fence, no cluster-wide barrier needed).
__device__ __forceinline__ void st_async_u64(uint32_t addr, u64 v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr), "l"(v),
                 "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, u64 a, u64 b, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "l"(a), "l"(b), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t mbar, uint32_t parity) {
    BW_STRESS(40);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(mbar), "r"(parity)
            : "memory");
    }
}

// Exchange transpose: registers of round RD (pre space) -> the post-space
// slots of the CTA that owns each element after the exchange.  The owner is
// given by the element's bits at positions P(i), which are register bits of
// round RD, so every destination is a compile-time choice per register.
// Elements staying in this CTA use plain shared stores; the others go out as
// st.async, which counts their bytes on the receiver's mbarrier.
template <class C, int RD, int RANK>
__device__ __forceinline__ void exchange_write_rank(const u64 (&v)[Dims<C>::E], u64* sm, uint32_t tp) {
    constexpr uint32_t pm = p_mask<C>();
    constexpr int NQ = 1 << C::Q;
    constexpr bool VEC = vec_smem<C, RD>();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t off =
        8u * (smem_slot_c<C>(to_local<C, C::XR>(tp)) + smem_slot_c<C>(to_local<C, C::XR>(RANK << kCtaBits)));
    const uint32_t mbar_local = sbase + 8u * Dims<C>::SMEM_ELEMS;
    uint32_t base[NQ], mbar[NQ];
#pragma unroll
    for (int d = 0; d < NQ; ++d) {
        base[d] = map_to_rank(sbase + off, (uint32_t)d);
        mbar[d] = map_to_rank(mbar_local, (uint32_t)d);
    }
    u64* local = sm + off / 8u;
    // Local stores first, then st.async to the partners (measured faster);
    // d is a compile-time value per register.  Vector rounds move pairs.
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
        for (int j = 0; j < Dims<C>::E; ++j) {
            if (VEC && (j & 1)) continue;
            const uint32_t rp = reg_part<C, RD>(j);
            uint32_t d = 0;
#pragma unroll
            for (int i = 0; i < C::Q; ++i) d |= ((rp >> C::P(i)) & 1u) << i;
            const uint32_t slot = smem_slot_c<C>(to_local<C, C::XR>(rp & ~pm));
            if (pass == 0 && d == (uint32_t)RANK) {
                if constexpr (VEC) {
                    ulonglong2 t;
                    t.x = v[j];
                    t.y = v[j + 1];
                    *reinterpret_cast<ulonglong2*>(local + slot) = t;
                } else {
                    local[slot] = v[j];
                }
            }
            if (pass == 1 && d != (uint32_t)RANK) {
                if constexpr (VEC)
                    st_async_v2(base[d] + 8u * slot, v[j], v[j + 1], mbar[d]);
                else
                    st_async_u64(base[d] + 8u * slot, v[j], mbar[d]);
            }
        }
    }
}

// Exchange transpose: registers of round RD (pre space) -> the post-space
// slots of the CTA that owns each element after the exchange.  The owner is
// given by the element's bits at positions P(i), which are register bits of
// round RD, so every destination is a compile-time choice per register; the
// code is specialised per cluster rank so no store needs a runtime branch.
// Elements staying in this CTA use plain shared stores; the others go out as
// st.async, which counts their bytes on the receiver's mbarrier.
template <class C, int RD>
__device__ __forceinline__ void exchange_write(const u64 (&v)[Dims<C>::E], u64* sm, uint32_t tp, uint32_t rank) {
    if constexpr (C::Q == 1) {
        if (rank == 0) exchange_write_rank<C, RD, 0>(v, sm, tp);
        else exchange_write_rank<C, RD, 1>(v, sm, tp);
    } else if constexpr (C::Q == 2) {
        switch (rank) {
            case 0: exchange_write_rank<C, RD, 0>(v, sm, tp); break;
            case 1: exchange_write_rank<C, RD, 1>(v, sm, tp); break;
            case 2: exchange_write_rank<C, RD, 2>(v, sm, tp); break;
            default: exchange_write_rank<C, RD, 3>(v, sm, tp); break;
        }
    }
}

template <class C, int L, int RD, bool FP = false>
__device__ __forceinline__ void run_rounds(u64 (&v)[Dims<C>::E], u64* sm, uint32_t lane, uint32_t warp,
                                           uint32_t rank, uint32_t parity = 0u) {
    if constexpr (RD < C::NR) {
        if constexpr (RD == C::XR) {
            static_assert((thread_part_bits<C, RD - 1>() & p_mask<C>()) == 0, "rank swap bits must be register bits");
            static_assert(RD == 1, "the DSMEM exchange is the first transpose (smem still unused)");
            // Partners have started (the arrive was issued right after the
            // loads); no smem has been read yet, so no WAR hazard exists.
            BW_STRESS(41);
            asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
            exchange_write<C, RD - 1>(v, sm, thread_part<C, RD - 1>(lane, warp), rank);
            BW_STRESS(42);
            __syncthreads();  // this CTA's own stores
            mbar_wait_parity((uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS), parity);  // remote bytes
        } else {
            BW_STRESS(43);
            if constexpr (RD > 1) __syncthreads();
            store_smem<C, RD - 1>(v, sm, thread_part<C, RD - 1>(lane, warp));
            BW_STRESS(44);
            __syncthreads();
        }
        BW_STRESS(45);
        load_smem<C, RD>(v, sm, thread_part<C, RD>(lane, warp));
        apply_stages<C, RD, L, FP>(v);
        run_rounds<C, L, RD + 1, FP>(v, sm, lane, warp, rank, parity);
    }
}

// Modes of the checked / restoring passes (k_pass's fused bound check,
// k_pass_map's compact plan).
enum { MAP_PLAIN = 0, MAP_CHECK = 1, MAP_RESTORE = 2 };

// Threshold extraction fused into the last pass (noisy.py:185-222 with
// |x| >= tau): the final register values are tested before the store and
// hits are appended (warp-aggregated) to an unordered list; bw_abi sorts
// the few hits by index afterwards.  count == nullptr disables it.
struct ExtractArgs {
    unsigned long long tau;
    unsigned long long base;  // index offset of element 0 (shards)
    long long* idx;
    long long* val;
    unsigned long long* count;
    unsigned long long cap;
};

__device__ __forceinline__ bool hit_ge_u(u64 x, unsigned long long tau) {
    const u64 mag = (long long)x < 0 ? (u64)0 - x : x;
    return mag >= tau;
}

// Any |v[j]| >= tau, in one add + one unsigned compare per element:
// |x| < tau  <=>  x + (tau - 1) in [0, 2 tau - 2] (mod 2^64), 1 <= tau <= 2^63.
template <int E>
__device__ __forceinline__ bool any_hit(const u64 (&v)[E], unsigned long long tau) {
    if (tau == 0) return true;
    if (tau > (1ull << 63)) return false;
    const u64 b = tau - 1, c = 2 * (tau - 1);
    bool any = false;
#pragma unroll
    for (int j = 0; j < E; ++j) any |= (v[j] + b) > c;
    return any;
}

// Slow path (a warp holds a hit): re-read the warp's just-stored values
// (the thread's own stores, program-ordered) so the registers of the tile
// are dead before the store; warp-aggregated append.  Out of line so the
// common path keeps the pass kernel's register budget.
template <class C, int RD, int T, int L>
__device__ __noinline__ void extract_slow(const u64* g, uint64_t gbase, uint32_t tp, int k, ExtractArgs ex) {
    constexpr int E = Dims<C>::E;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t t0 = global_off<T, L, SplitOf<C>::value>(tp, k);
#pragma unroll 1
    for (int j = 0; j < E; ++j) {
        const uint64_t off = t0 + global_off<T, L, SplitOf<C>::value>(reg_part<C, RD>(j), k);
        const u64 x = g[off];
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

// Cheap prefilter: OR over the registers of (x ^ sign(x)) (= |x| for x >= 0,
// |x| - 1 below), 3 instructions per value against any_hit's 5.  If that OR
// is below 2^p with 2^p <= tau - 1, every |x| <= 2^p <= tau - 1: no hit.
template <int E>
__device__ __forceinline__ bool maybe_hit(const u64 (&v)[E], unsigned long long tau) {
    if (tau < 2) return true;  // tau 0 / 1: (almost) everything hits, test exactly
    uint32_t ahi = 0, alo = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const uint32_t hi = (uint32_t)(v[j] >> 32), lo = (uint32_t)v[j];
        const uint32_t sg = (uint32_t)((int32_t)hi >> 31);
        ahi |= hi ^ sg;
        alo |= lo ^ sg;
    }
    const u64 acc = ((u64)ahi << 32) | alo;
    const int p = 63 - __clzll((long long)(tau - 1));  // 2^p <= tau - 1
    return (acc >> p) != 0;
}

template <class C, int RD, int T, int L>
__device__ __forceinline__ void extract_hits(const u64 (&v)[Dims<C>::E], const u64* g, uint64_t gbase, uint32_t tp,
                                             int k, const ExtractArgs& ex) {
    if (!__any_sync(0xffffffffu, maybe_hit<Dims<C>::E>(v, ex.tau))) return;  // the common case: no value near tau
    if (!__any_sync(0xffffffffu, any_hit<Dims<C>::E>(v, ex.tau))) return;    // exact: no hit in this warp
    extract_slow<C, RD, T, L>(g, gbase, tp, k, ex);
}

// One pass over every tile: load (round 0 layout) -> stages -> [transpose ->
// stages]* -> store (last round layout).  k = first global stage bit of the
// rows; for a low pass (L == T) the L2 prefetch distance in tiles (0: none).  Cluster configs (Q > 0) put 2^Q CTAs on one
// tile; grid = 2^(n-13) CTAs for every config.  SB > 0: the loads read a
// narrow SB-byte source `src` (widening first pass), the stores go to data.
//
// MODE (the low pass of fwht_inplace with the magnitude bound fused in,
// bw_fwht_inplace_i64; int64, no extraction, no narrow source):
//   MAP_CHECK: ex.tau = lim, ex.count = the abort word, ex.idx = the tile
//     flags.  A CTA that finds the abort word set skips its loads; every
//     input is tested against |x| <= lim (= 2^(63-n) - 1, core.py:80-94);
//     the CTAs of a cluster agree (DSMEM flags + one more cluster barrier);
//     a tile stores and sets its flag only if none of it is bad, else it
//     stores nothing and sets the abort word.
//   MAP_RESTORE: tiles without a flag exit; the others apply the same stages
//     again and shift right by ex.tau (H H = 2^w I): the input comes back.
template <class C, int L, bool EX = false, int SB = 0, bool FP = false, int MODE = MAP_PLAIN>
__global__ void __launch_bounds__(Dims<C>::NT, C::MINB)
    k_pass(u64* __restrict__ data, int k, ExtractArgs ex, const void* __restrict__ src) {
    static_assert(!SplitOf<C>::value, "split-row configs launch k_pass_split");
    static_assert(MODE == MAP_PLAIN || (L >= C::T && !EX && SB == 0 && !FP), "checked / restore: int64 low passes");
    constexpr int T = C::T;
    constexpr int E = Dims<C>::E;
    extern __shared__ u64 sm[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    uint64_t tile = blockIdx.x;
    if constexpr (C::Q > 0) tile = blockIdx.x >> C::Q;
    if constexpr (MODE == MAP_RESTORE) {
        if (*reinterpret_cast<volatile unsigned*>(reinterpret_cast<unsigned*>(ex.idx) + tile) == 0u) return;
    }
    if constexpr (C::Q > 0) rank = cluster_ctarank();
    u64* g = data + tile_base<T, L>(tile, k);

    if constexpr (C::Q > 0) {
        // mbarrier counting the bytes the partners will deliver to this CTA;
        // made visible cluster-wide before the (relaxed) cluster arrive.
        if (threadIdx.x == 0) {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS);
            constexpr uint32_t bytes_in = 8u * (Dims<C>::CTA - Dims<C>::CTA / Dims<C>::CLUSTER);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes_in) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    u64 v[E];
    [[maybe_unused]] bool skip = false, bad = false;
    if constexpr (MODE == MAP_CHECK) {
        skip = __syncthreads_or(threadIdx.x == 0 && *reinterpret_cast<volatile unsigned long long*>(ex.count) != 0ull);
        if (skip) {
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = 0;
        }
    }
    if (MODE == MAP_CHECK && skip) {
        // another tile failed the bound: keep the cluster in step, touch nothing
    } else if constexpr (SB > 0)
        load_global_narrow<C, 0, T, L, SB>(v, reinterpret_cast<const typename NarrowType<SB>::one*>(src) + tile_base<T, L>(tile, k),
                                           thread_part<C, 0>(lane, warp) | rank_bits<C, 0>(rank), k);
    else
        load_global<C, 0, T, L>(v, g, thread_part<C, 0>(lane, warp) | rank_bits<C, 0>(rank), k);
    if constexpr (L >= T && SB == 0) {
        // Low pass: k is an L2 prefetch distance in tiles (0 = none).  One
        // bulk prefetch of this CTA's 64 KB of the tile k launches ahead, so
        // that tile's loads find their lines in L2.
        if (k > 0 && threadIdx.x == 0) {
            const uint64_t pt = tile + (uint64_t)k;
            if (pt < (uint64_t)(gridDim.x >> C::Q)) {
                const u64* pp = data + (pt << T) + ((uint64_t)rank << kCtaBits);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pp), "r"(8u << kCtaBits) : "memory");
            }
        }
    }
    BW_STRESS(46);
    if constexpr (C::Q > 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    if constexpr (MODE == MAP_CHECK) {
        // |x| <= lim  <=>  x + lim in [0, 2 lim] (mod 2^64)
        const u64 lim = ex.tau, span = 2 * ex.tau;
        bad = skip;
#pragma unroll
        for (int j = 0; j < E; ++j) bad |= (v[j] + lim) > span;
    }
    apply_stages<C, 0, L, FP>(v);
    run_rounds<C, L, 1, FP>(v, sm, lane, warp, rank);
    constexpr int LAST = C::NR - 1;
    const uint32_t tp_last = thread_part<C, LAST>(lane, warp) | rank_bits<C, LAST>(rank);
    if constexpr (MODE == MAP_RESTORE) {
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = (u64)((long long)v[j] >> (int)ex.tau);
    }
    if constexpr (MODE == MAP_CHECK) {
        bool tile_bad = __syncthreads_or(bad);
        if constexpr (C::Q > 0) {
            const uint32_t fl = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS + 1);
            if (threadIdx.x == 0) {
#pragma unroll
                for (uint32_t d = 0; d < (uint32_t)Dims<C>::CLUSTER; ++d)
                    if (d != rank)
                        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(map_to_rank(fl + 8u * rank, d)),
                                     "l"((u64)tile_bad)
                                     : "memory");
            }
            BW_STRESS(56);
            cluster_sync_all();
#pragma unroll
            for (uint32_t d = 0; d < (uint32_t)Dims<C>::CLUSTER; ++d)
                if (d != rank) tile_bad |= reinterpret_cast<volatile u64*>(sm + Dims<C>::SMEM_ELEMS + 1)[d] != 0ull;
        }
        if (tile_bad) {
            if (threadIdx.x == 0 && !skip) atomicExch(ex.count, 1ull);
            return;
        }
        if (threadIdx.x == 0 && rank == 0) reinterpret_cast<unsigned*>(ex.idx)[tile] = 1u;
    }
    BW_STRESS(47);
    store_global<C, LAST, T, L>(v, g, tp_last, k);
    if constexpr (EX) extract_hits<C, LAST, T, L>(v, g, tile_base<T, L>(tile, k), tp_last, k, ex);
}

// Split-row pass (k = bw::split_pack(k, a, k2)): k_pass with the global
// loads and stores driven by the per-register offsets in the kernel's
// parameter space.  (A separate body, not a flag on k_pass: routing k_pass
// through a shared device function perturbed its register allocation and
// cost the 9-stage pass 1%, tools/gpu_ab.sh.)
//
// A > 0: the low run's length is the compile-time A, and every offset is
// computed like k_pass's (col + low rows << k + high rows << k2, the row
// parts compile-time per register) instead of read from the table: the
// table version keeps all 32 64-bit addresses live before the first load
// (128 registers) and ran 8-9% under its access-pattern walk at n = 34.
template <int T, int L, int A>
__device__ __forceinline__ uint64_t split_off_ct(uint32_t e, int k1, int k2) {
    const uint64_t col = e & ((1u << L) - 1u);
    const uint32_t row = e >> L;
    return col + ((uint64_t)(row & ((1u << A) - 1u)) << k1) + ((uint64_t)(row >> A) << k2);
}

template <class C, int L, bool EX = false, int A = 0>
__global__ void __launch_bounds__(Dims<C>::NT, C::MINB)
    k_pass_split(u64* __restrict__ data, int k, ExtractArgs ex, const __grid_constant__ SplitTab tab) {
    static_assert(SplitOf<C>::value && L < C::T, "k_pass_split takes split-row high-pass configs");
    constexpr int T = C::T;
    constexpr int E = Dims<C>::E;
    extern __shared__ u64 sm[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    uint64_t tile = blockIdx.x;
    if constexpr (C::Q > 0) {
        rank = cluster_ctarank();
        tile = blockIdx.x >> C::Q;
    }
    u64* g = data + tile_base<T, L, true>(tile, k);

    if constexpr (C::Q > 0) {
        // mbarrier counting the bytes the partners will deliver to this CTA;
        // made visible cluster-wide before the (relaxed) cluster arrive.
        if (threadIdx.x == 0) {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS);
            constexpr uint32_t bytes_in = 8u * (Dims<C>::CTA - Dims<C>::CTA / Dims<C>::CLUSTER);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes_in) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    u64 v[E];
    const uint32_t tp0 = thread_part<C, 0>(lane, warp) | rank_bits<C, 0>(rank);
    [[maybe_unused]] const int k1 = split_k(k), k2 = split_k2(k);
    if constexpr (A > 0) {
        const u64* p = g + split_off_ct<T, L, A>(tp0, k1, k2);
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = ld_pass(p + split_off_ct<T, L, A>(reg_part<C, 0>(j), k1, k2));
    } else {
        load_global_tab<C, T, L>(v, g, tp0, k, tab);
    }
    BW_STRESS(48);
    if constexpr (C::Q > 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    apply_stages<C, 0, L>(v);
    run_rounds<C, L, 1>(v, sm, lane, warp, rank);
    constexpr int LAST = C::NR - 1;
    const uint32_t tp_last = thread_part<C, LAST>(lane, warp) | rank_bits<C, LAST>(rank);
    BW_STRESS(49);
    if constexpr (A > 0) {
        u64* p = g + split_off_ct<T, L, A>(tp_last, k1, k2);
#pragma unroll
        for (int j = 0; j < E; ++j) st_pass(p + split_off_ct<T, L, A>(reg_part<C, LAST>(j), k1, k2), v[j]);
    } else {
        store_global_tab<C, T, L>(v, g, tp_last, k, tab);
    }
    if constexpr (EX) extract_hits<C, LAST, T, L>(v, g, tile_base<T, L, true>(tile, k), tp_last, k, ex);
}

// ---------------------------------------------------------------------------
// Mapped passes (the narrow-intermediate transform, bw_fwht_i64_narrow):
// k_pass's rounds, but the source and the destination each have their own
// element type and their own LAYOUT -- a permutation of the index bits (the
// natural order, or "tile-major for pass Q": pass Q's tiles stored one
// after another, tile-local index inside).  So a pass can write its output
// narrow (int16 / int32) and already in the order its successor reads,
// which then loads each tile as one contiguous block.  Offsets are linear
// over disjoint bits: per-register offsets (host table), per tile bit of
// the thread / cluster-rank part, and runs of tile-id bits per CTA.
// ---------------------------------------------------------------------------
struct LayoutTab {
    unsigned long long reg[32];  // offset of register index j (its tile bits) in the round
    unsigned long long bit[16];  // offset of virtual tile bit b
    int nruns;                   // tile id -> offset: sum of ((t >> src) & (2^len - 1)) << dst
    int rsrc[6], rlen[6], rdst[6];
};
struct MapArgs {
    LayoutTab ld, st;
    long long lim;  // stores narrower than 8 bytes: every |v| <= lim, else *flag |= 1
    // compact in-place plan (bw_fwht_i64_compact): MAP_CHECK passes test
    // every INPUT against lim, a tile writes only if its whole tile passed
    // and no tile has aborted (then tileflag[tile] = 1); MAP_RESTORE passes
    // run only on tiles with tileflag set and shift the result right.
    unsigned* tileflag;
    unsigned* abort;
    int shift;
};


template <typename T>
struct PairOf;
template <>
struct PairOf<short> {
    typedef short2 type;
};
template <>
struct PairOf<int> {
    typedef int2 type;
};
template <>
struct PairOf<long long> {
    typedef longlong2 type;
};

__device__ __forceinline__ unsigned long long layout_base(const LayoutTab& t, uint64_t tile, uint32_t vt) {
    unsigned long long off = 0;
#pragma unroll 1
    for (int r = 0; r < t.nruns; ++r) off += ((tile >> t.rsrc[r]) & ((1ull << t.rlen[r]) - 1ull)) << t.rdst[r];
#pragma unroll
    for (int b = 0; b < 16; ++b)
        if ((vt >> b) & 1u) off += t.bit[b];
    return off;
}

// TPC tiles per CTA (per cluster): every tile's loads are issued before the
// first tile is computed -- TPC times the bytes in flight, which narrow
// sources need to keep the load phase as long as an int64 one.  On cluster
// tiles each further tile re-arms the exchange mbarrier (phase u) and
// passes one more cluster barrier (the partner's shared memory is free).
//
// MODE (the compact in-place plan, bw_fwht_i64_compact; TPC = 1):
//   MAP_CHECK: a CTA that finds *abort set skips its loads; every input is
//     tested against |x| <= lim; the CTAs of a cluster agree through DSMEM
//     flags and one more cluster barrier; a tile stores (and sets
//     tileflag[tile]) only if no CTA of it is bad, else it stores nothing and
//     sets *abort.  So every tile either wrote its narrow output or left its
//     int64 input untouched.  Dynamic shared memory: + 8 B per cluster CTA.
//   MAP_RESTORE: tiles whose tileflag is 0 exit at once (uniformly per
//     cluster); the others shift their final values right by m.shift.
template <class C, int L, typename ST, typename DT, int TPC = 1, int MODE = MAP_PLAIN>
__global__ void __launch_bounds__(Dims<C>::NT, C::MINB)
    k_pass_map(const ST* __restrict__ src, DT* __restrict__ dst, unsigned* flag, const __grid_constant__ MapArgs m) {
    static_assert(MODE == MAP_PLAIN || TPC == 1, "check / restore passes hold one tile per CTA");
    constexpr int E = Dims<C>::E, LAST = C::NR - 1;
    extern __shared__ u64 sm[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    uint64_t tile = (uint64_t)blockIdx.x * TPC;
    if constexpr (C::Q > 0) tile = (uint64_t)(blockIdx.x >> C::Q) * TPC;
    if constexpr (MODE == MAP_RESTORE) {
        if (*reinterpret_cast<volatile unsigned*>(m.tileflag + tile) == 0u) return;  // the same for every CTA of the tile
    }
    if constexpr (C::Q > 0) {
        rank = cluster_ctarank();
        if (threadIdx.x == 0) {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS);
            constexpr uint32_t bytes_in = 8u * (Dims<C>::CTA - Dims<C>::CTA / Dims<C>::CLUSTER);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes_in) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    const uint32_t tp0 = thread_part<C, 0>(lane, warp) | rank_bits<C, 0>(rank);
    bool skip = false;  // MAP_CHECK: another tile already failed, this one only keeps the cluster in step
    if constexpr (MODE == MAP_CHECK)
        skip = __syncthreads_or(threadIdx.x == 0 && *reinterpret_cast<volatile unsigned*>(m.abort) != 0u);
    ST raw[TPC][E];
#pragma unroll
    for (int u = 0; u < TPC; ++u) {
        if constexpr (MODE == MAP_CHECK) {
            if (skip) {
#pragma unroll
                for (int j = 0; j < E; ++j) raw[u][j] = 0;
                continue;
            }
        }
        const ST* p = src + layout_base(m.ld, tile + u, tp0);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if constexpr (VecAccess<C, 0, L>::value) {  // tile bit 0 is offset bit 0 in every layout
                if ((j & 1) == 0) {
                    const typename PairOf<ST>::type t = ld_any(reinterpret_cast<const typename PairOf<ST>::type*>(p + m.ld.reg[j]));
                    raw[u][j] = t.x;
                    raw[u][j + 1] = t.y;
                }
            } else {
                raw[u][j] = ld_any(p + m.ld.reg[j]);
            }
        }
    }
    BW_STRESS(50);
    if constexpr (C::Q > 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    bool bad = false;
    if constexpr (MODE == MAP_CHECK) {
        bad = skip;
#pragma unroll
        for (int j = 0; j < E; ++j) bad |= ((long long)raw[0][j] > m.lim) | ((long long)raw[0][j] < -m.lim);
    }
#pragma unroll
    for (int u = 0; u < TPC; ++u) {
        u64 v[E];
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = (u64)(long long)raw[u][j];
        if (u > 0) {
            if constexpr (C::Q > 0) {
                if (threadIdx.x == 0) {  // phase u of the exchange mbarrier
                    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS);
                    constexpr uint32_t bytes_in = 8u * (Dims<C>::CTA - Dims<C>::CTA / Dims<C>::CLUSTER);
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes_in) : "memory");
                }
                // this CTA's reads of tile u-1 are done (release); run_rounds waits
                // for the partner's before writing into its shared memory
                BW_STRESS(51);
                asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
            } else {
                __syncthreads();  // the previous tile's last shared-memory reads
            }
        }
        apply_stages<C, 0, L>(v);
        run_rounds<C, L, 1>(v, sm, lane, warp, rank, (uint32_t)(u & 1));
        if constexpr (MODE == MAP_PLAIN && sizeof(DT) == 2) {  // the int32 stage after it cannot overflow (bw_fwht_i64_narrow)
#pragma unroll
            for (int j = 0; j < E; ++j) bad |= ((long long)v[j] > m.lim) | ((long long)v[j] < -m.lim);
        }
        if constexpr (MODE == MAP_RESTORE) {
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = (u64)((long long)v[j] >> m.shift);
        }
        if constexpr (MODE == MAP_CHECK) {
            // Tile-wide agreement: every CTA of the cluster stores, or none.
            bool tile_bad = __syncthreads_or(bad);
            if constexpr (C::Q > 0) {
                const uint32_t fl = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS + 1);
                if (threadIdx.x == 0) {
#pragma unroll
                    for (uint32_t d = 0; d < (uint32_t)Dims<C>::CLUSTER; ++d)
                        if (d != rank) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(map_to_rank(fl + 8u * rank, d)),
                                                    "l"((u64)tile_bad)
                                                    : "memory");
                }
                BW_STRESS(52);
                cluster_sync_all();
#pragma unroll
                for (uint32_t d = 0; d < (uint32_t)Dims<C>::CLUSTER; ++d)
                    if (d != rank) tile_bad |= reinterpret_cast<volatile u64*>(sm + Dims<C>::SMEM_ELEMS + 1)[d] != 0ull;
            }
            if (tile_bad) {
                if (threadIdx.x == 0 && !skip) atomicExch(m.abort, 1u);
                return;
            }
            if (threadIdx.x == 0 && rank == 0) m.tileflag[tile] = 1u;
        }
        DT* q = dst + layout_base(m.st, tile + u, thread_part<C, LAST>(lane, warp) | rank_bits<C, LAST>(rank));
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if constexpr (VecAccess<C, LAST, L>::value) {
                if ((j & 1) == 0) {
                    typename PairOf<DT>::type t;
                    t.x = (DT)(long long)v[j];
                    t.y = (DT)(long long)v[j + 1];
                    st_pass(reinterpret_cast<typename PairOf<DT>::type*>(q + m.st.reg[j]), t);
                }
            } else {
                st_pass(q + m.st.reg[j], (DT)(long long)v[j]);
            }
        }
    }
    if constexpr (MODE == MAP_PLAIN && sizeof(DT) == 2) {
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1u);
    }
}

// ---------------------------------------------------------------------------
// Small transforms (n <= 21): both passes of a two-pass plan in ONE
// cooperative launch -- every CTA transforms its low-bits tile, the grid
// synchronises (gpu-scope fences; each element was written by exactly one
// CTA), then every CTA runs its high-bits tile.  Saves a launch and the
// inter-kernel drain on the latency-bound sizes.  Single-CTA configs only.
// ---------------------------------------------------------------------------
template <class C, int L, bool FP>
__device__ __forceinline__ void single_tile(u64* __restrict__ data, int k, uint64_t tile, u64* sm) {
    static_assert(C::Q == 0, "single-CTA tiles only");
    constexpr int T = C::T, E = Dims<C>::E, LAST = C::NR - 1;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    u64* g = data + tile_base<T, L, SplitOf<C>::value>(tile, k);
    u64 v[E];
    load_global<C, 0, T, L>(v, g, thread_part<C, 0>(lane, warp), k);
    apply_stages<C, 0, L, FP>(v);
    run_rounds<C, L, 1, FP>(v, sm, lane, warp, 0u);
    store_global<C, LAST, T, L>(v, g, thread_part<C, LAST>(lane, warp), k);
}

template <class C1, int L1, class C2, int L2, bool FP = false>
__global__ void __launch_bounds__(256, 1) k_two_pass(u64* __restrict__ data, int k2) {
    extern __shared__ u64 sm[];
    single_tile<C1, L1, FP>(data, 0, blockIdx.x, sm);
    BW_STRESS(53);
    __syncthreads();  // shared memory is reused by the second tile
    cooperative_groups::this_grid().sync();
    single_tile<C2, L2, FP>(data, k2, blockIdx.x, sm);
}

// Sort the (few) fused-extraction hits by index in place: one CTA, bitonic
// in shared memory, count <= 2048.
__global__ void __launch_bounds__(1024) k_sort_hits(long long* idx, long long* val, const unsigned long long* count) {
    __shared__ long long sk[2048], sv[2048];
    const unsigned long long c = *count;
    const unsigned m = c < 2048ull ? (unsigned)c : 2048u;  // callers sort only when count <= 2048
    for (unsigned i = threadIdx.x; i < 2048; i += blockDim.x) {
        sk[i] = i < m ? idx[i] : 0x7FFFFFFFFFFFFFFFll;
        sv[i] = i < m ? val[i] : 0;
    }
    __syncthreads();
    for (unsigned size = 2; size <= 2048; size <<= 1) {
        for (unsigned stride = size >> 1; stride > 0; stride >>= 1) {
            for (unsigned i = threadIdx.x; i < 2048; i += blockDim.x) {
                const unsigned jx = i ^ stride;
                if (jx > i) {
                    const bool up = (i & size) == 0;
                    if ((sk[i] > sk[jx]) == up) {
                        const long long a = sk[i], b = sv[i];
                        sk[i] = sk[jx];
                        sv[i] = sv[jx];
                        sk[jx] = a;
                        sv[jx] = b;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (unsigned i = threadIdx.x; i < m; i += blockDim.x) {
        idx[i] = sk[i];
        val[i] = sv[i];
    }
}

// ---------------------------------------------------------------------------
template <typename S>
__global__ void k_widen(const S* __restrict__ src, long long* __restrict__ dst, uint64_t count) {
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += nth) dst[i] = src[i];
}

// Small transforms (n <= 13) and the float64 low-bits tiles: each CTA owns a
// contiguous 2^n tile in shared memory and applies stages 0..n-1 in
// ascending order (the order of core.py:108, which float64 bit identity
// needs; for int64 any order is exact).
// ---------------------------------------------------------------------------
template <typename V>
__global__ void __launch_bounds__(256) k_small(V* __restrict__ data, int n) {
    extern __shared__ __align__(16) unsigned char sm_raw[];
    V* sm = reinterpret_cast<V*>(sm_raw);
    const uint32_t N = 1u << n;
    V* d = data + (uint64_t)blockIdx.x * N;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) sm[i] = d[i];
    __syncthreads();
    for (int k = 0; k < n; ++k) {
        const uint32_t low = (1u << k) - 1u;
        for (uint32_t t = threadIdx.x; t < (N >> 1); t += blockDim.x) {
            const uint32_t lo = ((t >> k) << (k + 1)) | (t & low);
            const uint32_t hi = lo + (1u << k);
            const V a = sm[lo], b = sm[hi];
            sm[lo] = a + b;
            sm[hi] = a - b;
        }
        __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) d[i] = sm[i];
}

// K0: one radix-2 stage k over the whole signal (Fig. 1 inner loop,
// PAPER.md:189-201; pairing formula of parallel.py:108).  Debug/reference
// aid for int64; the high stages of the float64 path.
template <typename V>
__global__ void k_stage(V* __restrict__ data, uint64_t half, int k) {
    const uint64_t low = (1ull << k) - 1ull;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < half;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = ((t >> k) << (k + 1)) | (t & low);
        const uint64_t hi = lo + (1ull << k);
        const V a = data[lo], b = data[hi];
        data[lo] = a + b;
        data[hi] = a - b;
    }
}

__global__ void k_scale_f64(double* __restrict__ data, uint64_t count, double f) {
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += nth) data[i] *= f;
}

// ---------------------------------------------------------------------------
// K3: max/min reduction (magnitude bound, core.py:80-94).
// ---------------------------------------------------------------------------
__global__ void k_minmax_init(long long* out) {
    out[0] = (long long)0x8000000000000000ull;  // running max starts at INT64_MIN
    out[1] = (long long)0x7FFFFFFFFFFFFFFFull;  // running min starts at INT64_MAX
}

// One CTA per contiguous 2^16-point chunk (like k_extract_count): enough
// CTAs for every SM to keep loads in flight to the end.  (A grid-stride loop
// over one wave of CTAs read at 2.5 TB/s, tools/aux_bench.py.)
constexpr int kMinmaxChunkBits = 16;
__global__ void __launch_bounds__(512) k_minmax(const long long* __restrict__ data, uint64_t count,
                                                long long* out) {
    long long mx = (long long)0x8000000000000000ull, mn = (long long)0x7FFFFFFFFFFFFFFFull;
    const uint64_t start = (uint64_t)blockIdx.x << kMinmaxChunkBits;
    const uint64_t end = min(count, start + (uint64_t)(1ull << kMinmaxChunkBits));
    const bool aligned = ((reinterpret_cast<uintptr_t>(data) & 15u) == 0);
    uint64_t done = start;
    if (aligned) {
        const longlong2* p = reinterpret_cast<const longlong2*>(data);
        const uint64_t p0 = start >> 1, p1 = end >> 1;
#pragma unroll 8
        for (uint64_t i = p0 + threadIdx.x; i < p1; i += blockDim.x) {
            const longlong2 a = __ldcs(p + i);
            mx = max(mx, max(a.x, a.y));
            mn = min(mn, min(a.x, a.y));
        }
        done = p1 << 1;
    }
    for (uint64_t i = done + threadIdx.x; i < end; i += blockDim.x) {
        const long long a = data[i];
        mx = max(mx, a);
        mn = min(mn, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    __shared__ long long smx[32], smn[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        smx[w] = mx;
        smn[w] = mn;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        mx = l < nw ? smx[l] : (long long)0x8000000000000000ull;
        mn = l < nw ? smn[l] : (long long)0x7FFFFFFFFFFFFFFFull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (l == 0) {
            atomicMax(&out[0], mx);
            atomicMin(&out[1], mn);
        }
    }
}

// ---------------------------------------------------------------------------
// K6: cross-shard P-point butterfly (parallel.py:103-110 stage phases, all
// log2 P of them fused; one pass over the P shards' slice).
// ---------------------------------------------------------------------------
struct ShardPtrs {
    u64* p[8];
};

template <int LOGP>
__global__ void __launch_bounds__(256) k_xshard(ShardPtrs s, uint64_t begin, uint64_t pairs) {
    constexpr int P = 1 << LOGP;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < pairs; q += nth) {
        const uint64_t i = begin + 2 * q;
        ulonglong2 v[P];
#pragma unroll
        for (int r = 0; r < P; ++r) v[r] = __ldcs(reinterpret_cast<const ulonglong2*>(s.p[r] + i));
#pragma unroll
        for (int b = 0; b < LOGP; ++b) {
#pragma unroll
            for (int r = 0; r < P; ++r) {
                if (!((r >> b) & 1)) {
                    const ulonglong2 a = v[r], c = v[r | (1 << b)];
                    v[r].x = a.x + c.x;
                    v[r].y = a.y + c.y;
                    v[r | (1 << b)].x = a.x - c.x;
                    v[r | (1 << b)].y = a.y - c.y;
                }
            }
        }
#pragma unroll
        for (int r = 0; r < P; ++r) __stcs(reinterpret_cast<ulonglong2*>(s.p[r] + i), v[r]);
    }
}

// ---------------------------------------------------------------------------
// Narrow-wire cross-shard stage: the log2 P cross stages run FIRST, on the
// untransformed input (stages on distinct bits commute in Z/2^64).  When
// every |x| <= lim = floor(WMAX / P) (WMAX = 127 for int8, 32767 for int16),
// every intermediate of the P-point butterfly satisfies |y| <= P * lim <=
// WMAX, so the shards are packed to W-byte integers, the exchange moves W
// bytes per point over NVLink instead of 8, and each device's local
// transform widens its packed shard in the first pass (bw_fwht_widen).
// ---------------------------------------------------------------------------
template <typename W>
struct WireWord;
template <>
struct WireWord<signed char> {  // 4 int8 lanes per 32-bit word
    static __device__ __forceinline__ unsigned add(unsigned a, unsigned b) { return __vadd4(a, b); }
    static __device__ __forceinline__ unsigned sub(unsigned a, unsigned b) { return __vsub4(a, b); }
};
template <>
struct WireWord<short> {  // 2 int16 lanes per 32-bit word
    static __device__ __forceinline__ unsigned add(unsigned a, unsigned b) { return __vadd2(a, b); }
    static __device__ __forceinline__ unsigned sub(unsigned a, unsigned b) { return __vsub2(a, b); }
};

// int64 -> W, 8 points per thread (64-byte read, 8W-byte write); *flag |= 1
// if some |x| > lim (the caller then takes the int64 path; x is unchanged).
template <typename W>
__global__ void __launch_bounds__(256) k_pack_narrow(const long long* __restrict__ x, W* __restrict__ out,
                                                     uint64_t count, long long lim, unsigned* flag) {
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < count / 8; q += nth) {
        const longlong2* src = reinterpret_cast<const longlong2*>(x + 8 * q);
        W w[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const longlong2 a = __ldcs(src + i);
            bad |= (a.x > lim) | (a.x < -lim) | (a.y > lim) | (a.y < -lim);
            w[2 * i] = (W)a.x;
            w[2 * i + 1] = (W)a.y;
        }
        if constexpr (sizeof(W) == 1) {
            uint2 o;
            o.x = (unsigned)(unsigned char)w[0] | (unsigned)(unsigned char)w[1] << 8 |
                  (unsigned)(unsigned char)w[2] << 16 | (unsigned)(unsigned char)w[3] << 24;
            o.y = (unsigned)(unsigned char)w[4] | (unsigned)(unsigned char)w[5] << 8 |
                  (unsigned)(unsigned char)w[6] << 16 | (unsigned)(unsigned char)w[7] << 24;
            *reinterpret_cast<uint2*>(out + 8 * q) = o;
        } else {
            uint4 o;
            o.x = (unsigned)(unsigned short)w[0] | (unsigned)(unsigned short)w[1] << 16;
            o.y = (unsigned)(unsigned short)w[2] | (unsigned)(unsigned short)w[3] << 16;
            o.z = (unsigned)(unsigned short)w[4] | (unsigned)(unsigned short)w[5] << 16;
            o.w = (unsigned)(unsigned short)w[6] | (unsigned)(unsigned short)w[7] << 16;
            *reinterpret_cast<uint4*>(out + 8 * q) = o;
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31u) == 0) atomicOr(flag, 1u);
}

struct NarrowPtrs {
    void* p[8];
};

// The P-point butterfly over elements [begin, begin + count) of the P packed
// shards (peer pointers), 16 bytes of every shard per thread, packed SIMD
// add/sub on the W-bit lanes (exact: no lane leaves the W range).
template <typename W, int LOGP>
__global__ void __launch_bounds__(256) k_xshard_narrow(NarrowPtrs s, uint64_t begin, uint64_t count) {
    constexpr int P = 1 << LOGP, PER = 16 / sizeof(W);
    typedef WireWord<W> WW;
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < count / PER; q += nth) {
        const uint64_t e = begin + q * PER;
        uint4 v[P];
#pragma unroll
        for (int r = 0; r < P; ++r) v[r] = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<W*>(s.p[r]) + e));
#pragma unroll
        for (int b = 0; b < LOGP; ++b) {
#pragma unroll
            for (int r = 0; r < P; ++r) {
                if (!((r >> b) & 1)) {
                    const uint4 a = v[r], c = v[r | (1 << b)];
                    v[r] = make_uint4(WW::add(a.x, c.x), WW::add(a.y, c.y), WW::add(a.z, c.z), WW::add(a.w, c.w));
                    v[r | (1 << b)] =
                        make_uint4(WW::sub(a.x, c.x), WW::sub(a.y, c.y), WW::sub(a.z, c.z), WW::sub(a.w, c.w));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < P; ++r) __stcs(reinterpret_cast<uint4*>(reinterpret_cast<W*>(s.p[r]) + e), v[r]);
    }
}

// ---------------------------------------------------------------------------
// K6': the last local high pass FUSED with the cross-shard stage.  The tile
// of a high pass (C::T bits, one CTA or a 2-CTA cluster) is split as L
// columns, r local rows at stride 2^k, and the top LOGP bits = the shard
// index: every CTA loads its tile rows from all P shards (peer pointers over
// NVLink), applies the r local stages AND the log2 P cross-shard stages, and
// stores back to every shard -- one kernel, compute and exchange fused.
// Each device runs the tiles [tile0, tile0 + gridDim.x / 2^Q); the devices'
// tile ranges are disjoint (the check_disjoint argument,
// parallel.py:114-134).  In the round-0 and last-round layouts the shard
// bits are register, warp or cluster-rank bits, so every shard-pointer
// lookup is warp-uniform.
// ---------------------------------------------------------------------------
template <class C, int L, int LOGP, bool EX = false>
__global__ void __launch_bounds__(Dims<C>::NT, C::MINB)
    k_pass_x(ShardPtrs s, int k, uint64_t tile0, ExtractArgs ex, int nl) {
    constexpr int T = C::T, E = Dims<C>::E, TL = T - LOGP, LAST = C::NR - 1;
    constexpr uint32_t lmask = (1u << TL) - 1u;
    extern __shared__ u64 sm[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    if constexpr (C::Q > 0) {
        rank = cluster_ctarank();
        if (threadIdx.x == 0) {
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(sm + Dims<C>::SMEM_ELEMS);
            constexpr uint32_t bytes_in = 8u * (Dims<C>::CTA - Dims<C>::CTA / Dims<C>::CLUSTER);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes_in) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    const uint64_t base = tile_base<TL, L>(tile0 + (blockIdx.x >> C::Q), k);  // within a shard
    u64 v[E];
    {
        const uint32_t tp = thread_part<C, 0>(lane, warp) | rank_bits<C, 0>(rank);
        const uint64_t t0 = base + global_off<TL, L>(tp & lmask, k);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const uint32_t e = reg_part<C, 0>(j);
            v[j] = ld_pass(s.p[(tp | e) >> TL] + t0 + global_off<TL, L>(e & lmask, k));
        }
    }
    BW_STRESS(54);
    if constexpr (C::Q > 0) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    apply_stages<C, 0, L>(v);
    run_rounds<C, L, 1>(v, sm, lane, warp, rank);
    const uint32_t tp = thread_part<C, LAST>(lane, warp) | rank_bits<C, LAST>(rank);
    const uint64_t t1 = base + global_off<TL, L>(tp & lmask, k);
    BW_STRESS(55);
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const uint32_t e = reg_part<C, LAST>(j);
        st_pass(s.p[(tp | e) >> TL] + t1 + global_off<TL, L>(e & lmask, k), v[j]);
    }
    // Fused extraction (configs 3/5 over several GPUs): |W| >= tau on the
    // final values, global index = shard << nl + offset, warp-aggregated
    // append (unordered; sorted afterwards).
    if constexpr (EX) {
        if (!__any_sync(0xffffffffu, maybe_hit<E>(v, ex.tau))) return;
        if (!__any_sync(0xffffffffu, any_hit<E>(v, ex.tau))) return;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const bool h = hit_ge_u(v[j], ex.tau);
            const unsigned b = __ballot_sync(0xffffffffu, h);
            if (!b) continue;
            const int leader = __ffs(b) - 1;
            unsigned long long first = 0;
            if ((int)lane == leader) first = atomicAdd(ex.count, (unsigned long long)__popc(b));
            first = __shfl_sync(0xffffffffu, first, leader);
            if (h) {
                const unsigned long long pos = first + __popc(b & ((1u << lane) - 1u));
                if (pos < ex.cap) {
                    const uint32_t e = reg_part<C, LAST>(j);
                    const uint64_t shard = (tp | e) >> TL;
                    ex.idx[pos] = (long long)(ex.base + (shard << nl) + t1 + global_off<TL, L>(e & lmask, k));
                    ex.val[pos] = (long long)v[j];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K4: seeded counter-based generators (oracle/oracle_np.py restates them).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
__host__ __device__ __forceinline__ uint64_t hash64(uint64_t seed, uint64_t i) {
    return fmix64((i * 0x9E3779B97F4A7C15ull) ^ seed);
}

struct GenParams {
    int kind;
    int nmasks;
    uint64_t seed;
    uint64_t a;    // UNIFORM: A
    uint64_t thr;  // NOISY: noise threshold
    uint64_t mask[8];
    uint64_t mseed[8];
};

__device__ __forceinline__ long long gen_value(const GenParams& g, uint64_t i) {
    if (g.kind == 1) return 1 - 2 * (long long)(hash64(g.seed, i) & 1ull);
    if (g.kind == 2) return (long long)(hash64(g.seed, i) % (2 * g.a + 1)) - (long long)g.a;
    long long x = 0;
    for (int m = 0; m < g.nmasks; ++m) {
        const uint64_t bit = (uint64_t)(__popcll(g.mask[m] & i) & 1) ^ (uint64_t)(hash64(g.mseed[m], i) < g.thr);
        x += 1 - 2 * (long long)bit;
    }
    return x;
}

__global__ void __launch_bounds__(256) k_gen(long long* __restrict__ out, uint64_t base, uint64_t count,
                                             GenParams g) {
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += nth)
        out[i] = gen_value(g, base + i);
}

// ---------------------------------------------------------------------------
// K5: ordered threshold extraction (noisy.py:185-222): |x| >= tau.
// Phase A counts hits per chunk, phase B scans the counts, phase C rewrites
// only the chunks that hold hits, in index order -- no sort needed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool hit_ge(long long x, uint64_t tau) {
    const uint64_t mag = x < 0 ? (uint64_t)0 - (uint64_t)x : (uint64_t)x;
    return mag >= tau;
}

constexpr int kExtractChunkBits = 16;

// Hit predicates of the extraction kernels (noisy.py:218 np.abs(x) >= tau).
struct HitI64 {
    uint64_t tau;
    __device__ __forceinline__ bool operator()(long long x) const { return hit_ge(x, tau); }
};
struct HitF64 {  // NaN never hits, like numpy's comparison
    double tau;
    __device__ __forceinline__ bool operator()(long long bits) const {
        return fabs(__longlong_as_double(bits)) >= tau;
    }
};

template <class H>
__global__ void __launch_bounds__(512) k_extract_count(const long long* __restrict__ data, uint64_t count,
                                                       H hit, unsigned long long* counts) {
    const uint64_t chunk = 1ull << kExtractChunkBits;
    const uint64_t start = blockIdx.x * chunk;
    const uint64_t end = min(count, start + chunk);
    unsigned c = 0;
    for (uint64_t i = start + threadIdx.x; i < end; i += blockDim.x) c += hit(__ldcs(data + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
        counts[blockIdx.x] = s;
    }
}

// Exclusive scan of counts[0..m) in place; total -> counts[m].  One CTA.
__global__ void __launch_bounds__(1024) k_extract_scan(unsigned long long* counts, uint64_t m) {
    __shared__ unsigned long long ws[32];
    __shared__ unsigned long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t base = 0; base < m; base += blockDim.x) {
        const uint64_t i = base + threadIdx.x;
        const unsigned long long x = i < m ? counts[i] : 0ull;
        unsigned long long incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (l >= o) incl += y;
        }
        if (l == 31) ws[w] = incl;
        __syncthreads();
        if (w == 0) {
            unsigned long long t = l < (int)(blockDim.x >> 5) ? ws[l] : 0ull;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
                if (l >= o) t += y;
            }
            ws[l] = t;  // inclusive prefix over warps
        }
        __syncthreads();
        const unsigned long long wpre = w > 0 ? ws[w - 1] : 0ull;
        if (i < m) counts[i] = carry + wpre + incl - x;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += ws[(blockDim.x >> 5) - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) counts[m] = carry;
}

template <class H>
__global__ void __launch_bounds__(512) k_extract_write(const long long* __restrict__ data, uint64_t count,
                                                       H hit, const unsigned long long* offsets,
                                                       const unsigned long long* counts_after,
                                                       uint64_t base_index, long long* out_idx,
                                                       long long* out_val, uint64_t cap) {
    const uint64_t chunk = 1ull << kExtractChunkBits;
    const uint64_t start = blockIdx.x * chunk;
    const unsigned long long off0 = offsets[blockIdx.x];
    if (counts_after[blockIdx.x] == off0) return;  // no hits in this chunk
    const uint64_t end = min(count, start + chunk);
    __shared__ unsigned ws[32];
    __shared__ unsigned long long running;
    if (threadIdx.x == 0) running = off0;
    __syncthreads();
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint64_t s = start; s < end; s += blockDim.x) {
        const uint64_t i = s + threadIdx.x;
        long long x = 0;
        bool h = false;
        if (i < end) {
            x = data[i];
            h = hit(x);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, h);
        if (l == 0) ws[w] = __popc(bal);
        __syncthreads();
        unsigned wpre = 0, tot = 0;
        for (int q = 0; q < nw; ++q) {
            const unsigned c = ws[q];
            wpre += q < w ? c : 0u;
            tot += c;
        }
        if (h) {
            const unsigned long long pos = running + wpre + __popc(bal & ((1u << l) - 1u));
            if (pos < cap) {
                out_idx[pos] = (long long)(base_index + i);
                out_val[pos] = x;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) running += tot;
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// wht_bruteforce (core.py:128-144): y_i = sum_j (-1)^popcount(i & j) x_j,
// O(4^n), out of place; the "oracle of the oracle" for n <= 14.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bruteforce(const long long* __restrict__ x, long long* __restrict__ y,
                                                    int n) {
    __shared__ long long xs[2048];
    const uint32_t N = 1u << n;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (uint32_t j0 = 0; j0 < N; j0 += 2048) {
        const uint32_t m = min(2048u, N - j0);
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < m; t += blockDim.x) xs[t] = x[j0 + t];
        __syncthreads();
        if (i < N)
            for (uint32_t t = 0; t < m; ++t) {
                const u64 v = (u64)xs[t];
                acc += (__popc(i & (j0 + t)) & 1) ? (u64)0 - v : v;
            }
    }
    if (i < N) y[i] = (long long)acc;
}

// parseval_energy (core.py:176-185), exact for int64: every thread sums x^2
// as a 192-bit integer (x^2 < 2^127), blocks write (lo, hi, top) partials.
// CTA b sums the contiguous range [b * chunk, (b + 1) * chunk) with 16-byte
// loads (contiguous ranges over many CTAs: every SM keeps loads in flight).
__global__ void __launch_bounds__(256) k_sumsq(const long long* __restrict__ x, uint64_t count,
                                               unsigned long long* partial) {
    unsigned __int128 acc = 0;
    unsigned long long top = 0;
    const uint64_t chunk = ((count + gridDim.x - 1) / gridDim.x + 1) & ~1ull;  // even
    const uint64_t start = min(count, (uint64_t)blockIdx.x * chunk), end = min(count, start + chunk);
    auto add = [&](long long v) {
        const unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
        const unsigned __int128 sq = (unsigned __int128)a * a;
        acc += sq;
        top += acc < sq;
    };
    uint64_t done = start;
    if ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
        const longlong2* p = reinterpret_cast<const longlong2*>(x);
#pragma unroll 4
        for (uint64_t i = (start >> 1) + threadIdx.x; i < (end >> 1); i += blockDim.x) {
            const longlong2 a = __ldcs(p + i);
            add(a.x);
            add(a.y);
        }
        done = (end >> 1) << 1;
        if (done < start) done = start;
    }
    for (uint64_t i = done + threadIdx.x; i < end; i += blockDim.x) add(x[i]);
    __shared__ unsigned long long s_lo[256], s_hi[256], s_top[256];
    s_lo[threadIdx.x] = (unsigned long long)acc;
    s_hi[threadIdx.x] = (unsigned long long)(acc >> 64);
    s_top[threadIdx.x] = top;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned __int128 sum = 0;
        unsigned long long t = 0;
        for (int k = 0; k < (int)blockDim.x; ++k) {
            const unsigned __int128 p = ((unsigned __int128)s_hi[k] << 64) | s_lo[k];
            sum += p;
            t += (sum < p) + s_top[k];
        }
        partial[3 * blockIdx.x + 0] = (unsigned long long)sum;
        partial[3 * blockIdx.x + 1] = (unsigned long long)(sum >> 64);
        partial[3 * blockIdx.x + 2] = t;
    }
}

// ---------------------------------------------------------------------------
// fold (subspace.py:150-161): out[L.j] += x[j] over j in [0, 2^d_in), where
// L.j is the XOR of the column masks of L selected by the bits of j
// (apply_map_array, subspace.py:116-121), looked up 8 index bits at a time.
// Small outputs (d_out <= 12) are accumulated per CTA in shared memory.
// x == nullptr folds the seeded generator's signal on the fly (no input).
// ---------------------------------------------------------------------------
constexpr int kFoldGroups = 5;  // d_in <= 40

template <bool SMEM_BINS, int NT = 256>
__global__ void __launch_bounds__(NT) k_fold(const long long* __restrict__ x, uint64_t count,
                                              const unsigned* __restrict__ table, int groups, int d_out,
                                              unsigned long long* out, GenParams g) {
    __shared__ unsigned tab[kFoldGroups * 256];
    // Shared bins as separate low / high 32-bit words: a 64-bit shared
    // atomicAdd compiles to a CAS loop, 32-bit ones are native.  The low
    // word's returned old value gives the exact carry into the high word,
    // so hi * 2^32 + lo is the exact sum mod 2^64.
    extern __shared__ unsigned bins32[];
    unsigned* lo = bins32;
    unsigned* hi = bins32 + (SMEM_BINS ? (1 << d_out) : 0);
    for (int i = threadIdx.x; i < groups * 256; i += blockDim.x) tab[i] = table[i];
    if (SMEM_BINS)
        for (int i = threadIdx.x; i < (2 << d_out); i += blockDim.x) bins32[i] = 0u;
    __syncthreads();
    const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
    auto add = [&](unsigned t, unsigned long long v) {
        if (SMEM_BINS) {
            const unsigned vl = (unsigned)v, vh = (unsigned)(v >> 32);
            const unsigned old = atomicAdd(&lo[t], vl);
            const unsigned carry = (old + vl) < old ? 1u : 0u;
            if (vh + carry) atomicAdd(&hi[t], vh + carry);
        } else {
            atomicAdd(&out[t], v);
        }
    };
    if (count >= 4) {
        // Quads of consecutive indices: L.j is linear, so L.(4m + i) =
        // L.(4m) ^ L.i -- one set of table lookups per four points, and two
        // 16-byte loads.
        const unsigned l1 = tab[1], l2 = tab[2], l3 = tab[3];
        const bool vec = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
        const uint64_t quads = count >> 2;
        for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < quads; m += nth) {
            const uint64_t j = m << 2;
            unsigned t = 0;
            for (int q = 0; q < groups; ++q) t ^= tab[q * 256 + ((j >> (8 * q)) & 255u)];
            unsigned long long v0, v1, v2, v3;
            if (x && vec) {
                const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(x + j);
                const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(x + j + 2);
                v0 = a.x, v1 = a.y, v2 = b.x, v3 = b.y;
            } else if (x) {  // 8-byte aligned view
                v0 = (unsigned long long)x[j], v1 = (unsigned long long)x[j + 1];
                v2 = (unsigned long long)x[j + 2], v3 = (unsigned long long)x[j + 3];
            } else {
                v0 = (unsigned long long)gen_value(g, j);
                v1 = (unsigned long long)gen_value(g, j + 1);
                v2 = (unsigned long long)gen_value(g, j + 2);
                v3 = (unsigned long long)gen_value(g, j + 3);
            }
            add(t, v0);
            add(t ^ l1, v1);
            add(t ^ l2, v2);
            add(t ^ l3, v3);
        }
    } else {
        for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count; j += nth) {
            unsigned t = 0;
            for (int q = 0; q < groups; ++q) t ^= tab[q * 256 + ((j >> (8 * q)) & 255u)];
            add(t, x ? (unsigned long long)x[j] : (unsigned long long)gen_value(g, j));
        }
    }
    if (SMEM_BINS) {
        __syncthreads();
        for (int i = threadIdx.x; i < (1 << d_out); i += blockDim.x) {
            const unsigned long long b = ((unsigned long long)hi[i] << 32) | lo[i];
            if (b) atomicAdd(&out[i], b);
        }
    }
}

// ---------------------------------------------------------------------------
// fold with d_out > 12 through a change of output basis (bw_abi fold_blocks):
// with the low K columns of L independent, an invertible A makes
//   u = A L j = (e ^ c(h)) | blk(h) << 14,   j = h * 2^14 + e,
// so every contiguous 2^14-point chunk h lands, permuted by XOR with c(h),
// on ONE block of 2^14 bins.  A CTA owns one block in shared memory and
// streams the chunks mapping to it (h = h0(b) ^ kernel combinations, each
// chunk 128 KB contiguous): no atomics while accumulating, 8 B/point of
// reads; the block is flushed to out[A^-1 u] at the end.
// ---------------------------------------------------------------------------
// Bins per CTA 2^12 (32 KB) on 512 threads, several CTAs per SM: measured
// best of 2^12..2^14 bins x 256..1024 threads (2^32 -> 2^20: 6.8 ms, against
// 8.2 for 2^13 x 512 and 9.4 for 2^14 x 1024; profiles/r01_fold_ab*.log).
#ifndef BW_FOLD_BITS
#define BW_FOLD_BITS 12
#endif
#ifndef BW_FOLD_THREADS
#define BW_FOLD_THREADS 512
#endif
constexpr int kFoldBlockBits = BW_FOLD_BITS;
constexpr int kFoldThreads = BW_FOLD_THREADS;

struct FoldBlockArgs {
    const long long* x;  // nullptr: the seeded generator's signal
    GenParams g;
    unsigned long long* out;
    const unsigned long long* h0;   // per image block: a chunk index mapping to it
    const unsigned* bval;           // per image block: its u >> 14
    const unsigned long long* kap;  // [4][256] XOR of kernel vectors by 8-bit groups of the chunk counter
    const unsigned* ftop;           // [4][256] c(h) by 8-bit groups of h
    const unsigned* bmap;           // [4][256] A^-1 u by 8-bit groups of u
    const unsigned* gtab;           // !INJ: in-block bin of chunk point e (2^K entries)
    int nsplit;                     // CTAs per block
    uint64_t nchunk;                // chunks per block
};

// !INJ (the default): bin = gtab[e] ^ c, the bins are 32-bit low / high
// words updated with native shared atomics and an exact carry, like
// k_fold's shared bins -- correct for any L (also dependent low columns,
// where points of one chunk share bins) and needs no barrier per chunk.
// INJ (BW_FOLD_PLAIN=1, independent low columns): a chunk's points land on
// distinct bins e ^ c, plain adds, one barrier per chunk (measured slower).
template <bool INJ>
__global__ void __launch_bounds__(kFoldThreads, 1024 / kFoldThreads) k_fold_blocks(FoldBlockArgs a) {
    extern __shared__ unsigned long long fsm[];
    constexpr int B = 1 << kFoldBlockBits;
    unsigned long long* acc = fsm;
    unsigned* lo = reinterpret_cast<unsigned*>(fsm);
    unsigned* hi = lo + B;
    unsigned long long* kap = fsm + B;
    unsigned* ftop = reinterpret_cast<unsigned*>(kap + 1024);
    unsigned* bmap = ftop + 1024;
    unsigned* gtab = bmap + 1024;  // !INJ only
    const int bi = blockIdx.x / a.nsplit, sp = blockIdx.x % a.nsplit;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        kap[i] = a.kap[i];
        ftop[i] = a.ftop[i];
        bmap[i] = a.bmap[i];
    }
    if constexpr (!INJ)
        for (int i = threadIdx.x; i < B; i += blockDim.x) gtab[i] = a.gtab[i];
    for (int i = threadIdx.x; i < B; i += blockDim.x) acc[i] = 0ull;
    __syncthreads();
    const uint64_t q0 = a.nchunk * sp / a.nsplit, q1 = a.nchunk * (sp + 1) / a.nsplit;
    const uint64_t h0 = a.h0[bi];
    auto chunk_of = [&](uint64_t q) {
        return h0 ^ kap[q & 255] ^ kap[256 + ((q >> 8) & 255)] ^ kap[512 + ((q >> 16) & 255)] ^
               kap[768 + ((q >> 24) & 255)];
    };
    auto c_of = [&](uint64_t h) {
        return ftop[h & 255] ^ ftop[256 + ((h >> 8) & 255)] ^ ftop[512 + ((h >> 16) & 255)] ^
               ftop[768 + ((h >> 24) & 255)];
    };
    constexpr int PER = B / kFoldThreads / 2;  // element pairs per thread per chunk
    ulonglong2 cur[PER], nxt[PER];
    auto load = [&](uint64_t h, ulonglong2 (&r)[PER]) {
        const uint64_t base = h << kFoldBlockBits;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const uint64_t e = 2u * threadIdx.x + 2u * kFoldThreads * i;
            if (a.x) {
                r[i] = __ldcs(reinterpret_cast<const ulonglong2*>(a.x + base + e));
            } else {
                r[i].x = (unsigned long long)gen_value(a.g, base + e);
                r[i].y = (unsigned long long)gen_value(a.g, base + e + 1);
            }
        }
    };
    if (q0 < q1) load(chunk_of(q0), cur);
    for (uint64_t q = q0; q < q1; ++q) {
        const uint32_t c = c_of(chunk_of(q));
        if (q + 1 < q1) load(chunk_of(q + 1), nxt);  // the next chunk's loads fly over this chunk's adds
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const uint32_t e = 2u * threadIdx.x + 2u * kFoldThreads * i;
            if constexpr (INJ) {
                const uint32_t p = e ^ c;  // e + 1 lands on p ^ 1
                acc[p] += cur[i].x;
                acc[p ^ 1u] += cur[i].y;
            } else {
                const unsigned long long vv[2] = {cur[i].x, cur[i].y};
#pragma unroll
                for (int w = 0; w < 2; ++w) {
                    const uint32_t t = gtab[e + w] ^ c;
                    const unsigned vl = (unsigned)vv[w], vh = (unsigned)(vv[w] >> 32);
                    const unsigned old = atomicAdd(&lo[t], vl);
                    const unsigned carry = (old + vl) < old ? 1u : 0u;
                    if (vh + carry) atomicAdd(&hi[t], vh + carry);
                }
            }
        }
        if constexpr (INJ) __syncthreads();  // the next chunk's permutation differs: its bins may be another thread's
#pragma unroll
        for (int i = 0; i < PER; ++i) cur[i] = nxt[i];
    }
    const unsigned b = a.bval[bi];
    if constexpr (!INJ) __syncthreads();
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
        const unsigned long long v = INJ ? acc[i] : ((unsigned long long)hi[i] << 32) | lo[i];
        if (!v) continue;
        const uint32_t u = (uint32_t)i | (b << kFoldBlockBits);
        const uint32_t t = bmap[u & 255] ^ bmap[256 + ((u >> 8) & 255)] ^ bmap[512 + ((u >> 16) & 255)] ^
                           bmap[768 + ((u >> 24) & 255)];
        if (a.nsplit == 1) a.out[t] = v;
        else atomicAdd(a.out + t, v);
    }
}

// ---------------------------------------------------------------------------
// Elementwise helpers for the inverse transform (core.py:147-173).
// ---------------------------------------------------------------------------
// One CTA per contiguous 2^16-point chunk with 16-byte accesses (as k_minmax).
__global__ void __launch_bounds__(512) k_check_divisible(const long long* __restrict__ data, uint64_t count, int n,
                                                         int* flag) {
    const uint64_t m = (1ull << n) - 1ull;
    const uint64_t start = (uint64_t)blockIdx.x << kMinmaxChunkBits;
    const uint64_t end = min(count, start + (uint64_t)(1ull << kMinmaxChunkBits));
    uint64_t bad = 0, done = start;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) == 0) {
        const ulonglong2* p = reinterpret_cast<const ulonglong2*>(data);
#pragma unroll 8
        for (uint64_t i = (start >> 1) + threadIdx.x; i < (end >> 1); i += blockDim.x) {
            const ulonglong2 a = __ldcs(p + i);
            bad |= (a.x | a.y) & m;  // Python % on ints: divisible iff the low n bits are 0
        }
        done = (end >> 1) << 1;
    }
    for (uint64_t i = done + threadIdx.x; i < end; i += blockDim.x) bad |= ((uint64_t)data[i]) & m;
    if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31u) == 0) *flag = 1;
}

__global__ void __launch_bounds__(512) k_shift_right(long long* __restrict__ data, uint64_t count, int n) {
    const uint64_t start = (uint64_t)blockIdx.x << kMinmaxChunkBits;
    const uint64_t end = min(count, start + (uint64_t)(1ull << kMinmaxChunkBits));
    uint64_t done = start;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) == 0) {
        longlong2* p = reinterpret_cast<longlong2*>(data);
#pragma unroll 8
        for (uint64_t i = (start >> 1) + threadIdx.x; i < (end >> 1); i += blockDim.x) {
            longlong2 a = p[i];
            a.x >>= n;  // exact division (floor == exact when divisible)
            a.y >>= n;
            p[i] = a;
        }
        done = (end >> 1) << 1;
    }
    for (uint64_t i = done + threadIdx.x; i < end; i += blockDim.x) data[i] = data[i] >> n;
}

}  // namespace bw
