// bw_abi.cu -- C ABI of the B200 FWHT (declared in include/bigwht_b200.h).
//
// Host-side planning, validation, launches and error mapping.  Every entry
// point cites the reference interface it replaces; see the header.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <math.h>
#include <string.h>

#include <stdlib.h>

#include <mutex>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/bigwht_b200.h"
#include "bw_kernels.cuh"
#include "bw_kernels32.cuh"
#include "bw_layouts.h"

using bw::u64;
typedef int CUresult_compat;

namespace {

thread_local std::string g_err;

int fail(int status, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return status;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(BW_CUDA_ERROR, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define BW_CUDA(call)                                  \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

#define BW_LAUNCHED(what)                                  \
    do {                                                   \
        cudaError_t e_ = cudaGetLastError();               \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

#define BW_TRY(expr)                  \
    do {                              \
        int s_ = (expr);              \
        if (s_ != BW_OK) return s_;   \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kMaxDevices = 64;
std::mutex g_mu;
bool g_attr_done[kMaxDevices];
int g_num_sms[kMaxDevices];
// BW_TWO_PASS=0 disables the single-launch path for two-pass plans (A/B knob).
const bool g_two_pass = !(getenv("BW_TWO_PASS") && getenv("BW_TWO_PASS")[0] == '0');
// BW_NARROW_TPC=1|2|4: tiles per CTA (or cluster) of the narrow plan's high passes (default 2,
// measured best: n = 32 in 30.4 ms against 31.6 with one tile; four spill).
const int g_narrow_tpc = getenv("BW_NARROW_TPC") ? atoi(getenv("BW_NARROW_TPC")) : 2;
// BW_SPLIT_CT=0: split-row passes read their offsets from the table (A/B knob).
const bool g_split_ct = !(getenv("BW_SPLIT_CT") && getenv("BW_SPLIT_CT")[0] == '0');
// BW_LOW_PREFETCH=<tiles>[,<tiles for clusters>]: the low passes bulk-prefetch into L2 the tile
// that many launches ahead (A/B knob; read per call).
int low_prefetch_tiles(int q) {
    const char* e = getenv("BW_LOW_PREFETCH");
    if (!e || !*e) return 0;
    const int a = atoi(e);
    const char* c = strchr(e, ',');
    return (q > 0 && c) ? atoi(c + 1) : a;
}
// BW_FUSED_BOUND=0: fwht_inplace runs the separate bound reduction first (A/B knob).
const bool g_fused_bound = !(getenv("BW_FUSED_BOUND") && getenv("BW_FUSED_BOUND")[0] == '0');
// BW_COMPACT (read per call): unset / "auto" -- fwht_array and fwht_inplace
// try the compact in-place plan where it measured faster than the int64 plan
// (compact_default below: every pass on the int32 engine, n = 30..32); "1" --
// wherever a compact plan exists (n >= 22); "0" -- never.
int compact_mode() {
    const char* e = getenv("BW_COMPACT");
    if (!e || !*e || e[0] == 'a') return -1;
    return e[0] == '1' ? 1 : 0;
}
bool compact_default(int log2n, const void* data);                       // after compact_plan
int compact_try(int64_t* data, int log2n, cudaStream_t s, int* used,
                const bw::ExtractArgs* ex = nullptr);  // after launch_compact
// BW_FOLD_BLOCKS=0 keeps the shared-bin / L2-atomic fold for d_out > 12 (A/B knob, read per call).
bool fold_blocks_enabled() { return !(getenv("BW_FOLD_BLOCKS") && getenv("BW_FOLD_BLOCKS")[0] == '0'); }
// BW_F64_VEC_LOW=0 keeps the float64 low pass on 8-byte accesses (A/B knob).
const bool g_f64_vec_low = !(getenv("BW_F64_VEC_LOW") && getenv("BW_F64_VEC_LOW")[0] == '0');
// BW_SPLIT_PLANS=0 keeps the default planner to one-run high passes (A/B knob).
const bool g_split_plans = !(getenv("BW_SPLIT_PLANS") && getenv("BW_SPLIT_PLANS")[0] == '0');
// BW_HOST_PIPELINE=0 disables the copy/compute overlap of host-buffer transforms (A/B knob).
const bool g_host_pipeline = !(getenv("BW_HOST_PIPELINE") && getenv("BW_HOST_PIPELINE")[0] == '0');
// Small device scratch (reduction results, extraction counts, fold tables)
// for calls that get none from the caller.  Per host thread: every call that
// uses it synchronises its stream before returning, so a thread never has two
// uses in flight, and calls from different threads never share a buffer.
struct ThreadScratch {
    void* p[kMaxDevices] = {};
    size_t bytes[kMaxDevices] = {};
};
thread_local ThreadScratch t_scratch;

int set_all_pass_attributes();

// Per-device one-time setup: opt-in dynamic shared memory sizes.
int device_setup(int* dev_out) {
    int dev = 0;
    BW_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= kMaxDevices) return fail(BW_NOT_SUPPORTED, "device id %d out of range", dev);
    *dev_out = dev;
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_attr_done[dev]) return BW_OK;
    int major = 0, minor = 0;
    BW_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    BW_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
    if (major != 10 || minor != 0)
        return fail(BW_NOT_SUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a (B200) only",
                    dev, major, minor);
    BW_CUDA(cudaDeviceGetAttribute(&g_num_sms[dev], cudaDevAttrMultiProcessorCount, dev));
    BW_TRY(set_all_pass_attributes());
    BW_CUDA(cudaFuncSetAttribute(bw::k_small<u64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (1 << 13) * 8));
    BW_CUDA(cudaFuncSetAttribute(bw::k_small<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (1 << 13) * 8));
    BW_CUDA(cudaFuncSetAttribute(bw::k_fold<true, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 << 14));
    g_attr_done[dev] = true;
    return BW_OK;
}

// Internal per-device scratch (never the signal itself).
int scratch(int dev, size_t bytes, void** out) {
    ThreadScratch& t = t_scratch;
    if (t.bytes[dev] < bytes) {
        if (t.p[dev]) cudaFree(t.p[dev]);  // the previous use on this thread has completed
        t.p[dev] = nullptr;
        t.bytes[dev] = 0;
        size_t want = bytes < 4096 ? 4096 : bytes;
        cudaError_t e = cudaMalloc(&t.p[dev], want);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(scratch)");
        t.bytes[dev] = want;
    }
    *out = t.p[dev];
    return BW_OK;
}

int grid_for(int dev, uint64_t work_items, int threads, int per_sm) {
    const uint64_t need = (work_items + threads - 1) / threads;
    const uint64_t cap = (uint64_t)g_num_sms[dev] * per_sm;
    uint64_t g = need < cap ? need : cap;
    return g < 1 ? 1 : (int)g;
}

// ---- pass plan -------------------------------------------------------------
//
// A plan is a list of pass widths: the low-bits pass (stages 0..w0-1 on
// contiguous tiles; w0 = 13, 14 or 15 uses a cluster of 1, 2 or 4 CTAs, and
// w0 = n <= 12 the single-CTA small kernel) followed by high-bits passes in
// ascending bit order.  A high width r picks its kernel: r <= 5 the
// register-only pass, r = 6..8 a single-CTA tile, r = 9 and 10 a cluster of 2
// (high_default_q; the measured planner below may pick other sizes).  Tests may
// force the cluster size of a high pass with the entry r | (q + 1) << 4.
//
// A high entry r | (q + 1) << 4 | a << 8 | k2 << 12 with a > 0 is a SPLIT
// pass (bw_layouts.h): its first a rows start at the lowest stage bit no
// earlier pass covered, the other r - a rows are bits [k2, k2 + r - a).
// A plain entry always starts at the lowest uncovered bit, so passes may
// come in any order (int64 stages commute); the plan must cover every bit
// exactly once.

enum PassKind { SMALL, LOW, HIGH, REG };

struct Pass {
    PassKind kind;
    int k;       // first stage bit
    int r;       // number of stages
    int q;       // log2 cluster size of LOW / HIGH passes
    int a = 0;   // split passes: rows [k, k+a) u [k2, k2+r-a); 0 = one run [k, k+r)
    int k2 = 0;
    // the kernels' int k argument (bw::split_pack for split passes)
    int karg() const { return a ? bw::split_pack(k, a, k2) : k; }
    // mask of the global stage bits of a LOW / HIGH / REG pass
    uint64_t stage_mask() const {
        if (kind == LOW) return (1ull << r) - 1ull;
        if (!a) return ((1ull << r) - 1ull) << k;
        return (((1ull << a) - 1ull) << k) | (((1ull << (r - a)) - 1ull) << k2);
    }
};

template <class T>
struct tag {
    using type = T;
};
template <int V>
using ic = std::integral_constant<int, V>;

// Calls f(tag<Cfg>, ic<L>) for the kernel instantiation L in [L, LMAX].
template <class C, int L, int LMAX, class F>
int with_L(int l, F& f) {
    if (l == L) return f(tag<C>{}, ic<L>{});
    if constexpr (L < LMAX) {
        return with_L<C, L + 1, LMAX>(l, f);
    } else {
        return fail(BW_BAD_ARGUMENTS, "no pass kernel instantiated for %d column bits", l);
    }
}

template <class F>
int visit_pass(const Pass& p, F&& f) {
    switch (p.kind) {
        case LOW:
            if (p.q == 0) return f(tag<bw::CfgLow13>{}, ic<13>{});
            if (p.q == 1) return f(tag<bw::CfgLow14c>{}, ic<14>{});
            return f(tag<bw::CfgLow15c>{}, ic<15>{});
        case HIGH:
            if (p.a > 0) {  // split rows: 6..8 rows on one CTA, 9..10 on a cluster of 2
                if (p.q == 0) return with_L<bw::CfgHigh13S, 5, 7>(13 - p.r, f);
                if (p.q == 1) return with_L<bw::CfgHigh14cS, 4, 5>(14 - p.r, f);
                return fail(BW_BAD_ARGUMENTS, "split rows need a cluster of 1 or 2");
            }
            if (p.q == 0) return with_L<bw::CfgHigh13, 3, 7>(13 - p.r, f);
            if (p.q == 1) return with_L<bw::CfgHigh14c, 4, 8>(14 - p.r, f);
            return with_L<bw::CfgHigh15c, 5, 10>(15 - p.r, f);
        case REG:
            return with_L<bw::CfgReg, 8, 12>(bw::CfgReg::T - p.r, f);
        default:
            return fail(BW_BAD_ARGUMENTS, "small transforms have no tile kernel");
    }
}

// Cluster size of a high pass when a plan entry does not force one (the
// out-of-core chunks and the fused multi-device plan): 9 and 10 stages run
// on a cluster of 2 (a 2^14 tile keeps 256-/128-byte row segments).
int high_default_q(int r) { return r <= 8 ? 0 : 1; }

// ---- measured cost model of the default planner --------------------------
// HBM TB/s of every pass shape the planner can emit, by the stage bit k the
// pass starts at (tools/sweep_shapes.py on one B200, profiles/r01_shapes_*;
// n = 32 and 34 agree to 1%: the rate depends on the row stride 2^k and the
// row-segment length, not on n).  A pass moves 16 B/point whatever its
// shape, so a plan's time is proportional to sum(1 / rate).
// generated by tools/gen_shape_table.py from profiles/r01_shapes_n34.json (NVIDIA B200)
// low passes 13 / 14 / 15 bits:
constexpr int kLowEff[3] = {702, 593, 450};
// rows: reg r=3,4,5; high r=6..10 x q=0,1.  columns: k = 13..31
constexpr int kShapeEff[13][19] = {
    {696, 695, 697, 696, 695, 677, 691, 685, 686, 687, 688, 688, 689, 689, 691, 690, 687, 687, 688},  // r=3 q=0
    {698, 698, 698, 696, 692, 690, 687, 681, 683, 683, 684, 686, 686, 686, 686, 684, 682, 684, 684},  // r=4 q=0
    {698, 698, 697, 693, 687, 685, 682, 679, 679, 680, 682, 684, 683, 682, 681, 672, 670, 670, 670},  // r=5 q=0
    {684, 697, 695, 678, 670, 664, 642, 619, 617, 632, 634, 625, 614, 602, 596, 603, 603, 603, 603},  // r=6 q=0
    {628, 626, 626, 621, 621, 619, 617, 616, 616, 618, 619, 618, 617, 618, 615, 608, 608, 608, 608},  // r=6 q=1
    {680, 684, 676, 646, 659, 639, 633, 650, 638, 644, 647, 629, 623, 605, 619, 619, 619, 619, 619},  // r=7 q=0
    {625, 624, 622, 624, 624, 621, 625, 622, 614, 616, 618, 623, 623, 622, 624, 624, 624, 624, 624},  // r=7 q=1
    {647, 642, 640, 645, 645, 634, 650, 643, 629, 639, 640, 602, 601, 589, 589, 589, 589, 589, 589},  // r=8 q=0
    {666, 653, 646, 647, 644, 654, 653, 646, 639, 652, 654, 654, 654, 645, 645, 645, 645, 645, 645},  // r=8 q=1
    {612, 610, 602, 602, 600, 588, 571, 564, 510, 511, 502, 500, 506, 506, 506, 506, 506, 506, 506},  // r=9 q=0
    {657, 639, 642, 641, 646, 649, 636, 613, 637, 643, 644, 646, 644, 644, 644, 644, 644, 644, 644},  // r=9 q=1
    {401, 397, 395, 383, 367, 360, 347, 331, 299, 299, 299, 299, 299, 299, 299, 299, 299, 299, 299},  // r=10 q=0
    {594, 612, 619, 626, 621, 615, 604, 583, 530, 530, 531, 531, 531, 531, 531, 531, 531, 531, 531},  // r=10 q=1
};

int shape_eff(int r, int q, int k) {
    const int kk = k < 13 ? 0 : k > 31 ? 18 : k - 13;
    if (r <= bw::kRegOnlyMaxBits) return kShapeEff[(r < 3 ? 3 : r) - 3][kk];
    return kShapeEff[3 + 2 * (r - 6) + q][kk];
}

// Cheapest split of stages [k0, k0 + h) into high passes (h / 10 rounded up
// passes, or one more), each with its best cluster shape at its k.  Returns
// the cost in units of 1e6 / (TB/s x 100); entries are r | (q + 1) << 4.
long long best_high_split(int k0, int h, std::vector<int>* out) {
    out->clear();
    if (h <= 0) return 0;
    const int m0 = (h + bw::kMaxHighBits - 1) / bw::kMaxHighBits;
    long long best = -1;
    std::vector<int> cur;
    // depth-first over compositions of h into m parts of 1..10
    struct Rec {
        static void go(int k, int left, int parts, long long cost, std::vector<int>& cur, std::vector<int>* out,
                       long long* best) {
            if (parts == 0) {
                if (left == 0 && (*best < 0 || cost < *best)) {
                    *best = cost;
                    *out = cur;
                }
                return;
            }
            for (int r = 1; r <= bw::kMaxHighBits && r <= left - (parts - 1); ++r) {
                if (left - r > (parts - 1) * bw::kMaxHighBits) continue;
                int entry = r, eff = shape_eff(r, 0, k);
                if (r > bw::kRegOnlyMaxBits) {
                    const int e1 = shape_eff(r, 1, k);
                    if (e1 > eff) {
                        eff = e1;
                        entry = r | (2 << 4);
                    } else {
                        entry = r | (1 << 4);
                    }
                }
                cur.push_back(entry);
                go(k + r, left - r, parts - 1, cost + 1000000 / eff, cur, out, best);
                cur.pop_back();
            }
        }
    };
    for (int m = m0; m <= m0 + 1 && m <= h; ++m) Rec::go(k0, h, m, 0, cur, out, &best);
    return best;
}

// BW_PLAN="13,10,9" overrides the default plan for a matching n
// (experiment knob; the checker and tests cover every legal plan).
bool env_plan(int n, std::vector<int>* widths) {
    const char* e = getenv("BW_PLAN");
    if (!e || !*e) return false;
    std::vector<int> w;
    int sum = 0;
    for (const char* c = e; *c;) {
        char* end = nullptr;
        const long v = strtol(c, &end, 10);
        if (end == c) return false;
        w.push_back((int)v);
        sum += (int)v & 15;
        c = (*end == ',') ? end + 1 : end;
    }
    if (w.empty() || sum - (w[0] & 15) + w[0] != n) return false;
    *widths = w;
    return true;
}

// Split-row passes on a cluster of 2 (9 or 10 rows: a low rows right above
// the low pass plus the top rows of the signal), TB/s x 100 by rows (9, 10)
// and a = 1..9.  Measured by tools/sweep_split.py at n = 32, 33, 34 with the
// compile-time-offset kernel (k_pass_split<..., A>; profiles/r02_split_n*.json,
// median over n and the low-pass width): the rate depends on a (how many rows
// share a DRAM page neighbourhood), not on n or on where the top run starts.
// (The offset-table kernel measured 5.52-5.83 for every a, r01_split_n*.json.)
constexpr int kSplitEff[2][10] = {
    {0, 648, 645, 615, 651, 640, 635, 645, 649, 0},     // 9 rows
    {0, 571, 602, 609, 619, 628, 630, 628, 624, 615}};  // 10 rows

// Three-pass plans with a split pass: low w0, the split pass (rows
// [w0, w0+a) u [n-(rs-a), n)), and one contiguous pass over the bits in
// between.  The contiguous pass is listed last, so a fused extraction runs
// on it.  Returns the cost (units as best_high_split) or -1.
long long best_split_plan(int n, int w0, std::vector<int>* out) {
    long long best = -1;
    for (int rs = 9; rs <= 10; ++rs) {
        const int rm = n - w0 - rs;
        if (rm < 1 || rm > bw::kMaxHighBits) continue;
        for (int a = 1; a < rs; ++a) {
            const int k2 = n - (rs - a), km = w0 + a;
            int em = shape_eff(rm, 0, km), entry = rm;
            if (rm > bw::kRegOnlyMaxBits) {
                const int e1 = shape_eff(rm, 1, km);
                if (e1 > em) {
                    em = e1;
                    entry = rm | (2 << 4);
                } else {
                    entry = rm | (1 << 4);
                }
            }
            if (!kSplitEff[rs - 9][a]) continue;
            const long long cost = 1000000 / kSplitEff[rs - 9][a] + 1000000 / em;
            if (best < 0 || cost < best) {
                best = cost;
                out->assign({rs | (2 << 4) | (a << 8) | (k2 << 12), entry});
            }
        }
    }
    return best;
}

// Default plan: the cheapest plan under the measured cost model (low pass
// of 13, 14 or 15 bits, then the best split of the rest into one-run high
// passes, or a split-row pass plus one contiguous pass).  Cached per n.
// one_run = true: only one-run high passes (the narrow plan's layouts have
// no split form).
int default_plan(int n, std::vector<int>* widths, bool one_run = false) {
    widths->clear();
    if (env_plan(n, widths)) return BW_OK;
    if (n == 0) return BW_OK;
    if (n <= 15) {
        widths->push_back(n);
        return BW_OK;
    }
    static std::mutex mu;
    static std::vector<int> cache[2][BW_MAX_LOG2N + 1];
    std::lock_guard<std::mutex> lock(mu);
    if (n <= BW_MAX_LOG2N && !cache[one_run][n].empty()) {
        *widths = cache[one_run][n];
        return BW_OK;
    }
    long long best_cost = -1;
    std::vector<int> hi;
    for (int w0 = 13; w0 <= 15 && w0 <= n; ++w0) {
        const long long cost = 1000000 / kLowEff[w0 - 13] + best_high_split(w0, n - w0, &hi);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            widths->assign(1, w0);
            widths->insert(widths->end(), hi.begin(), hi.end());
        }
        if (g_split_plans && !one_run && n >= 32) {  // measured at n = 32..34 (profiles/r02_split_n*.json)
            const long long sc = best_split_plan(n, w0, &hi);
            if (sc >= 0 && 1000000 / kLowEff[w0 - 13] + sc < best_cost) {
                best_cost = 1000000 / kLowEff[w0 - 13] + sc;
                widths->assign(1, w0);
                widths->insert(widths->end(), hi.begin(), hi.end());
            }
        }
    }
    if (n <= BW_MAX_LOG2N) cache[one_run][n] = *widths;
    return BW_OK;
}

int build_passes(int n, const std::vector<int>& widths, std::vector<Pass>* passes, bool partial = false) {
    passes->clear();
    if (n == 0) {
        if (!widths.empty()) return fail(BW_BAD_ARGUMENTS, "n = 0 takes no passes");
        return BW_OK;
    }
    if (widths.empty()) return fail(BW_BAD_ARGUMENTS, "empty pass plan for n = %d", n);
    const int w0 = widths[0];
    if (n <= 12) {
        if (w0 != n || widths.size() != 1)
            return fail(BW_BAD_ARGUMENTS, "a transform of n = %d <= 12 is one small pass", n);
        passes->push_back({SMALL, 0, n, 0});
        return BW_OK;
    }
    if (w0 < 13 || w0 > 15 || w0 > n)
        return fail(BW_BAD_ARGUMENTS, "the low pass covers 13, 14 or 15 bits (got %d, n = %d)", w0, n);
    passes->push_back({LOW, 0, w0, w0 - 13});
    uint64_t covered = (1ull << w0) - 1ull;
    for (size_t i = 1; i < widths.size(); ++i) {
        const int e = widths[i];
        const int r = e & 15;
        const int forced = ((e >> 4) & 15) - 1;
        const int a = (e >> 8) & 15, k2 = (e >> 12) & 63;
        if (e < 0 || (e >> 18) || r < 1 || r > bw::kMaxHighBits || forced > bw::kMaxClusterLog2 || a >= r)
            return fail(BW_BAD_ARGUMENTS, "bad high pass entry %d (width 1..%d, cluster q 0..%d, split 0..r-1)", e,
                        bw::kMaxHighBits, bw::kMaxClusterLog2);
        const int k = __builtin_ctzll(~covered);  // lowest uncovered bit
        Pass p;
        if (r <= bw::kRegOnlyMaxBits && forced <= 0 && a == 0) {
            p = {REG, k, r, 0};
        } else {
            const int q = forced >= 0 ? forced : high_default_q(r);
            const int L = 13 + q - r;
            const int lmin = q == 0 ? 3 : q == 1 ? 4 : 5;
            if (L < lmin || L > (q == 0 ? 7 : q == 1 ? 8 : 10))
                return fail(BW_BAD_ARGUMENTS, "no high-pass kernel for %d stages on a cluster of %d", r, 1 << q);
            p = {HIGH, k, r, q};
            if (a > 0) {
                if (k2 < k + a || (q == 0 ? (r < 6 || r > 8) : (q != 1 || r < 9)))
                    return fail(BW_BAD_ARGUMENTS, "bad split pass: rows [%d,%d) + [%d,%d) on a cluster of %d", k,
                                k + a, k2, k2 + r - a, 1 << q);
                p.a = a;
                p.k2 = k2;
            }
        }
        const uint64_t m = p.stage_mask();
        if (k + (a ? a : r) > 63 || (a && k2 + r - a > 63) || (m & covered))
            return fail(BW_BAD_ARGUMENTS, "high pass entry %d overlaps earlier passes", e);
        covered |= m;
        passes->push_back(p);
    }
    const uint64_t all = n >= 64 ? ~0ull : (1ull << n) - 1ull;
    if (covered & ~all) return fail(BW_BAD_ARGUMENTS, "pass widths reach beyond the signal's %d bits", n);
    if (covered != all && !(partial && covered == ((1ull << __builtin_ctzll(~covered)) - 1ull)))
        return fail(BW_BAD_ARGUMENTS, "pass widths cover %d of the signal's %d bits", __builtin_popcountll(covered), n);
    return BW_OK;
}

// Every kernel the planner can emit, for one-time setup.
template <class F>
int for_all_pass_kernels(F&& f) {
    for (int q = 0; q <= bw::kMaxClusterLog2; ++q) {
        BW_TRY(visit_pass(Pass{LOW, 0, 13 + q, q}, f));
        for (int L = (q == 0 ? 3 : q == 1 ? 4 : 5); L <= (q == 0 ? 7 : q == 1 ? 8 : 10); ++L)
            BW_TRY(visit_pass(Pass{HIGH, 0, 13 + q - L, q}, f));
    }
    for (int r = 1; r <= bw::kRegOnlyMaxBits; ++r) BW_TRY(visit_pass(Pass{REG, 0, r, 0}, f));
    for (int r = 6; r <= 10; ++r) {  // split-row variants
        Pass p{HIGH, 0, r, r <= 8 ? 0 : 1};
        p.a = 1;
        BW_TRY(visit_pass(p, f));
    }
    return BW_OK;
}

// ---- float64 passes (ascending stage order, CfgLow13F / CfgHigh13F / CfgReg)
template <class F>
int visit_pass_f64(const Pass& p, F&& f, bool vec = true) {
    switch (p.kind) {
        case LOW:
            if (vec && g_f64_vec_low) return f(tag<bw::CfgLow13FV>{}, ic<13>{});  // 16-byte aligned data
            return f(tag<bw::CfgLow13F>{}, ic<13>{});
        case HIGH:
            if (p.r == 8) return f(tag<bw::CfgHigh13F<5>>{}, ic<5>{});
            if (p.r == 7) return f(tag<bw::CfgHigh13F<6>>{}, ic<6>{});
            if (p.r == 6) return f(tag<bw::CfgHigh13F<7>>{}, ic<7>{});
            if (p.r == 9) return f(tag<bw::CfgHigh14cF<5>>{}, ic<5>{});
            if (p.r == 10) return f(tag<bw::CfgHigh14cF<4>>{}, ic<4>{});
            break;
        case REG:
            return with_L<bw::CfgReg, 8, 12>(bw::CfgReg::T - p.r, f);
        default:
            break;
    }
    return fail(BW_BAD_ARGUMENTS, "no float64 pass kernel for %d stages", p.r);
}

// float64 plan: one small pass (n <= 12), or the 13-bit low pass and then
// high passes of <= 10 stages in ascending bit order (9 and 10 stages on
// 2-CTA cluster tiles).
constexpr int kF64MaxHigh = 10;
int f64_passes(int n, std::vector<Pass>* passes) {
    passes->clear();
    if (n <= 0) return BW_OK;
    if (n <= 12) {
        passes->push_back({SMALL, 0, n, 0});
        return BW_OK;
    }
    passes->push_back({LOW, 0, 13, 0});
    const int h = n - 13;
    const int m = (h + kF64MaxHigh - 1) / kF64MaxHigh;
    int k = 13;
    for (int i = 0; i < m; ++i) {
        const int r = h / m + (i < h % m ? 1 : 0);
        passes->push_back({r <= bw::kRegOnlyMaxBits ? REG : HIGH, k, r, 0});
        k += r;
    }
    return BW_OK;
}

template <class F>
int for_all_f64_pass_kernels(F&& f) {
    BW_TRY(visit_pass_f64(Pass{LOW, 0, 13, 0}, f, true));
    BW_TRY(visit_pass_f64(Pass{LOW, 0, 13, 0}, f, false));
    for (int r = 1; r <= kF64MaxHigh; ++r)
        BW_TRY(visit_pass_f64(Pass{r <= bw::kRegOnlyMaxBits ? REG : HIGH, 0, r, 0}, f));
    return BW_OK;
}

template <int LOGP, int L>
int set_fused_attr() {
    if constexpr (L + LOGP <= 12) {
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_x<bw::CfgHigh13, L, LOGP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bw::Dims<bw::CfgHigh13>::SMEM_BYTES));
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_x<bw::CfgHigh13, L, LOGP, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, bw::Dims<bw::CfgHigh13>::SMEM_BYTES));
    }
    if constexpr (L >= 4 && L <= 8 && L + LOGP <= 13) {
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_x<bw::CfgHigh14c, L, LOGP>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bw::Dims<bw::CfgHigh14c>::SMEM_BYTES));
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_x<bw::CfgHigh14c, L, LOGP, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bw::Dims<bw::CfgHigh14c>::SMEM_BYTES));
    }
    return BW_OK;
}
template <int LOGP>
int set_fused_attrs() {
    BW_TRY((set_fused_attr<LOGP, 3>()));
    BW_TRY((set_fused_attr<LOGP, 4>()));
    BW_TRY((set_fused_attr<LOGP, 5>()));
    BW_TRY((set_fused_attr<LOGP, 6>()));
    BW_TRY((set_fused_attr<LOGP, 7>()));
    BW_TRY((set_fused_attr<LOGP, 8>()));
    BW_TRY((set_fused_attr<LOGP, 9>()));
    BW_TRY((set_fused_attr<LOGP, 10>()));
    BW_TRY((set_fused_attr<LOGP, 11>()));
    return BW_OK;
}

template <class C2, int L2>
int set_two_pass_attr() {
    constexpr int smem = bw::Dims<bw::CfgLow13>::SMEM_BYTES > bw::Dims<C2>::SMEM_BYTES ? bw::Dims<bw::CfgLow13>::SMEM_BYTES
                                                                                     : bw::Dims<C2>::SMEM_BYTES;
    BW_CUDA(cudaFuncSetAttribute(bw::k_two_pass<bw::CfgLow13, 13, C2, L2, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return BW_OK;
}

// k_pass_split with a compile-time low-run length A: dynamic shared memory
// attributes for every A (1 <= A < rows).
template <class C, int L, int A>
int split_ct_attributes(int smem) {
    if constexpr (A < C::T - L) {
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_split<C, L, false, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        BW_CUDA(cudaFuncSetAttribute(bw::k_pass_split<C, L, true, A>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        return split_ct_attributes<C, L, A + 1>(smem);
    }
    return BW_OK;
}

int set_all_pass_attributes() {
    for (int r = 1; r <= 8; ++r) {
        const Pass p{r <= bw::kRegOnlyMaxBits ? REG : HIGH, 13, r, 0};
        BW_TRY(visit_pass(p, [](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            if constexpr (C::Q == 0 && L < C::T && !bw::SplitOf<C>::value) return set_two_pass_attr<C, L>();
            return BW_OK;
        }));
    }
    // the int32 engine of the compact plan (64 KiB of shared memory, 2 CTAs/SM)
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_high<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_high<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_high<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_high<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_low<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_low<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_first<5, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_first<5, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_first<6, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_first<6, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_restore<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_CUDA(cudaFuncSetAttribute(bw::w32::k32_restore<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::w32::kSmemBytes));
    BW_TRY(set_fused_attrs<1>());
    BW_TRY(set_fused_attrs<2>());
    BW_TRY(set_fused_attrs<3>());
    BW_TRY(for_all_f64_pass_kernels([](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        constexpr int L = decltype(l)::value;
        constexpr int smem = bw::Dims<C>::SMEM_BYTES;
        if (smem > 48 * 1024) {
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false, false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        }
        return BW_OK;
    }));
    return for_all_pass_kernels([](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        constexpr int L = decltype(l)::value;
        constexpr int smem = bw::Dims<C>::SMEM_BYTES;
        if constexpr (bw::SplitOf<C>::value) {
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass_split<C, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass_split<C, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            if constexpr (C::Q == 1) {
                const int rc_ = split_ct_attributes<C, L, 1>(smem);
                if (rc_ != BW_OK) return rc_;
            }
        } else if (smem > 48 * 1024) {
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            if constexpr (L >= C::T) {  // widening low passes (int32 / int16 / int8 sources)
                BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem));
                BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem));
                BW_CUDA(cudaFuncSetAttribute(bw::k_pass<C, L, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem));
            }
        }
        return BW_OK;
    });
}

// Launch `kern` on `grid` CTAs of config C's shape (threads, dynamic shared
// memory) -- as thread-block clusters of C's size when C::Q > 0.
template <class C, class... KArgs, class... Args>
int launch_cfg(void (*kern)(KArgs...), unsigned grid, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(bw::Dims<C>::NT);
    cfg.dynamicSmemBytes = bw::Dims<C>::SMEM_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = bw::Dims<C>::CLUSTER;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = C::Q > 0 ? 1 : 0;
    BW_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
    return BW_OK;
}

// k_pass_split with the low-run length a as a compile-time A (1 <= A <
// rows), by recursion over A.
template <class C, int L, int A>
int launch_split_ct(int a, bool extract, unsigned grid, cudaStream_t s, u64* d, int karg, bw::ExtractArgs ex,
                    const bw::SplitTab& tab) {
    if constexpr (A < C::T - L) {
        if (a == A)
            return launch_cfg<C>(extract ? bw::k_pass_split<C, L, true, A> : bw::k_pass_split<C, L, false, A>, grid, s,
                                 d, karg, ex, tab);
        return launch_split_ct<C, L, A + 1>(a, extract, grid, s, d, karg, ex, tab);
    }
    return fail(BW_BAD_ARGUMENTS, "split pass with a = %d low rows", a);
}

// Element offsets of every register index in the load and the store round
// of a split-row pass (k_pass_split reads them from its parameters).
template <class C, int L>
bw::SplitTab split_table(int karg) {
    static_assert(bw::Dims<C>::E == 32, "32 registers per thread");
    constexpr int LAST = C::NR - 1;
    bw::SplitTab t;
    for (int j = 0; j < 32; ++j) {
        t.ld[j] = bw::global_off<C::T, L, true>(bw::reg_part<C, 0>(j), karg);
        t.st[j] = bw::global_off<C::T, L, true>(bw::reg_part<C, LAST>(j), karg);
    }
    return t;
}

// src != nullptr: the (low) pass reads a narrow source of src_bytes-byte
// integers and writes the int64 result to d (widening first pass).
int launch_pass(const Pass& p, u64* d, int n, cudaStream_t s, const bw::ExtractArgs* exp = nullptr,
                const void* src = nullptr, int src_bytes = 0) {
    bw::ExtractArgs ex = {};
    if (exp) ex = *exp;
    if (src && p.kind != LOW) return fail(BW_BAD_ARGUMENTS, "only the low pass widens a narrow input");
    if (src && src_bytes != 1 && src_bytes != 2 && src_bytes != 4)
        return fail(BW_BAD_ARGUMENTS, "narrow sources are 1, 2 or 4 bytes per point (got %d)", src_bytes);
    if (p.kind == SMALL) {
        bw::k_small<u64><<<1, 256, (size_t)(8ull << n), s>>>(d, n);
        BW_LAUNCHED("k_small launch");
        return BW_OK;
    }
    return visit_pass(p, [&](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        constexpr int L = decltype(l)::value;
        const unsigned grid = (unsigned)(1ull << (n - bw::kCtaBits));
        constexpr bool kLow = L >= C::T;
        const void* none = nullptr;
        if constexpr (bw::SplitOf<C>::value) {
            const bw::SplitTab tab = split_table<C, L>(p.karg());
            if constexpr (C::Q == 1) {  // compile-time low-run length (no offset table)
                if (g_split_ct && p.a >= 1 && p.a < C::T - L)
                    return launch_split_ct<C, L, 1>(p.a, ex.count != nullptr, grid, s, d, p.karg(), ex, tab);
            }
            if (ex.count) return launch_cfg<C>(bw::k_pass_split<C, L, true>, grid, s, d, p.karg(), ex, tab);
            return launch_cfg<C>(bw::k_pass_split<C, L, false>, grid, s, d, p.karg(), ex, tab);
        } else {
            if constexpr (kLow) {
                if (src && src_bytes == 4) return launch_cfg<C>(bw::k_pass<C, L, false, 4>, grid, s, d, p.k, ex, src);
                if (src && src_bytes == 2) return launch_cfg<C>(bw::k_pass<C, L, false, 2>, grid, s, d, p.k, ex, src);
                if (src) return launch_cfg<C>(bw::k_pass<C, L, false, 1>, grid, s, d, p.k, ex, src);
            }
            // low passes: k carries the L2 prefetch distance (BW_LOW_PREFETCH, tiles)
            const int karg = kLow ? low_prefetch_tiles(C::Q) : p.k;
            if constexpr (std::is_same_v<C, bw::CfgLow14c>) {
                static const bool minb3 = getenv("BW_LOW14_MINB3") && getenv("BW_LOW14_MINB3")[0] == '1';
                if (minb3 && !ex.count) {
                    auto kern = bw::k_pass<bw::CfgLow14c3, 14, false>;
                    BW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 bw::Dims<bw::CfgLow14c3>::SMEM_BYTES));
                    return launch_cfg<bw::CfgLow14c3>(kern, grid, s, d, karg, ex, none);
                }
            }
            if (ex.count) return launch_cfg<C>(bw::k_pass<C, L, true>, grid, s, d, karg, ex, none);
            return launch_cfg<C>(bw::k_pass<C, L, false>, grid, s, d, karg, ex, none);
        }
    });
}

int run_naive(u64* d, int n, int dev, cudaStream_t s) {
    const uint64_t half = n ? (1ull << (n - 1)) : 0;
    for (int k = 0; k < n; ++k) {
        bw::k_stage<u64><<<grid_for(dev, half, 256, 8), 256, 0, s>>>(d, half, k);
        BW_LAUNCHED("k_stage launch");
    }
    return BW_OK;
}

int check_signal(const void* data, int log2n) {
    if (log2n < 0 || log2n > BW_MAX_LOG2N)
        return fail(BW_BAD_ARGUMENTS, "log2n = %d outside 0..%d", log2n, BW_MAX_LOG2N);
    if (!data) return fail(BW_BAD_ARGUMENTS, "null signal pointer");
    if (reinterpret_cast<uintptr_t>(data) & 7u)
        return fail(BW_BAD_ARGUMENTS, "signal pointer is not 8-byte aligned");
    return BW_OK;
}

// Two-pass plans of single-CTA kernels whose grid fits on the GPU at once
// (n = 16..20 by default): one cooperative launch of k_two_pass.  Returns
// BW_OK with *done = false when the shape or the residency does not allow it.
int launch_two_pass(const std::vector<Pass>& passes, u64* d, int n, int dev, cudaStream_t s, bool* done) {
    *done = false;
    if (passes.size() != 2 || passes[0].kind != LOW || passes[0].q != 0 || passes[1].q != 0 || passes[1].a) return BW_OK;
    if (passes[1].kind != HIGH && passes[1].kind != REG) return BW_OK;
    const unsigned grid = 1u << (n - bw::kCtaBits);
    return visit_pass(passes[1], [&](auto t, auto l) -> int {
        using C2 = typename decltype(t)::type;
        constexpr int L2 = decltype(l)::value;
        if constexpr (C2::Q == 0 && L2 < C2::T && !bw::SplitOf<C2>::value) {
            auto kern = bw::k_two_pass<bw::CfgLow13, 13, C2, L2, false>;
            constexpr int smem = bw::Dims<bw::CfgLow13>::SMEM_BYTES > bw::Dims<C2>::SMEM_BYTES
                                     ? bw::Dims<bw::CfgLow13>::SMEM_BYTES
                                     : bw::Dims<C2>::SMEM_BYTES;
            int per_sm = 0;
            BW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
            if ((long long)per_sm * g_num_sms[dev] < (long long)grid) return BW_OK;
            int k2 = passes[1].k;
            void* args[] = {&d, &k2};
            BW_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(256), args, smem, s));
            *done = true;
        }
        return BW_OK;
    });
}

// The ascending-order layouts (8-byte accesses only): the float64 transform
// (FP) and int64 views that are 8- but not 16-byte aligned.
template <bool FP>
int run_scalar_plan(u64* d, int log2n, cudaStream_t s) {
    const bool vec = !(reinterpret_cast<uintptr_t>(d) & 15u);  // the paired low pass needs 16-byte alignment
    std::vector<Pass> passes;
    BW_TRY(f64_passes(log2n, &passes));
    for (const Pass& p : passes) {
        if (p.kind == SMALL) {
            if constexpr (FP)
                bw::k_small<double><<<1, 256, (size_t)(8ull << log2n), s>>>(reinterpret_cast<double*>(d), log2n);
            else
                bw::k_small<u64><<<1, 256, (size_t)(8ull << log2n), s>>>(d, log2n);
            BW_LAUNCHED("k_small launch");
            continue;
        }
        BW_TRY(visit_pass_f64(p, [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            const unsigned grid = (unsigned)(1ull << (log2n - bw::kCtaBits));
            const void* none = nullptr;
            return launch_cfg<C>(bw::k_pass<C, L, false, false, FP>, grid, s, d, p.k, bw::ExtractArgs{}, none);
        }, vec));
    }
    return BW_OK;
}

int fwht_impl(int64_t* data, int log2n, const std::vector<int>* widths, bool naive, cudaStream_t s) {
    BW_TRY(check_signal(data, log2n));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    u64* d = reinterpret_cast<u64*>(data);
    if (log2n == 0) return BW_OK;
    if (naive) return run_naive(d, log2n, dev, s);
    // 16-byte vector accesses need a 16-byte aligned base; an 8-byte aligned
    // view (e.g. an odd-offset slice) takes the 8-byte-access layouts.
    if (log2n >= bw::kCtaBits && (reinterpret_cast<uintptr_t>(data) & 15u)) return run_scalar_plan<false>(d, log2n, s);
    std::vector<int> w;
    if (widths) w = *widths; else BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    if (!widths && g_two_pass) {
        bool done = false;
        BW_TRY(launch_two_pass(passes, d, log2n, dev, s, &done));
        if (done) return BW_OK;
    }
    for (const Pass& p : passes) BW_TRY(launch_pass(p, d, log2n, s));
    return BW_OK;
}

uint64_t butterfly_count(int n) { return n == 0 ? 0 : (uint64_t)n << (n - 1); }

// Stages [lo, n) of a device buffer only (lo >= 13), through high passes:
// the out-of-core mode's device chunk holds 2^(n-lo) rows of 2^lo columns.
int fwht_high_bits(u64* d, int n, int lo, cudaStream_t s) {
    const int h = n - lo;
    if (h <= 0) return BW_OK;
    if (lo < bw::kCtaBits) return fail(BW_BAD_ARGUMENTS, "high-bit transform needs lo >= %d", bw::kCtaBits);
    std::vector<int> split;
    best_high_split(lo, h, &split);
    int k = lo;
    for (int e : split) {
        const int r = e & 15, q = (e >> 4) - 1;
        const Pass p = r <= bw::kRegOnlyMaxBits ? Pass{REG, k, r, 0} : Pass{HIGH, k, r, q};
        BW_TRY(launch_pass(p, d, n, s));
        k += r;
    }
    return BW_OK;
}



int minmax_impl(const int64_t* data, uint64_t count, int64_t* out, int dev, cudaStream_t s) {
    bw::k_minmax_init<<<1, 1, 0, s>>>(reinterpret_cast<long long*>(out));
    BW_LAUNCHED("k_minmax_init launch");
    (void)dev;
    const uint64_t grid = (count + (1ull << bw::kMinmaxChunkBits) - 1) >> bw::kMinmaxChunkBits;
    if (grid == 0) return BW_OK;
    bw::k_minmax<<<(unsigned)grid, 512, 0, s>>>(reinterpret_cast<const long long*>(data), count,
                                               reinterpret_cast<long long*>(out));
    BW_LAUNCHED("k_minmax launch");
    return BW_OK;
}

// M = max(max, -min) as an exact unsigned value; bound M * 2^n < 2^63.
uint64_t magnitude(int64_t mx, int64_t mn) {
    const uint64_t a = mx > 0 ? (uint64_t)mx : 0;
    const uint64_t b = mn < 0 ? (uint64_t)0 - (uint64_t)mn : 0;
    return a > b ? a : b;
}
bool bound_ok(uint64_t M, int n) {
    if (M == 0) return true;
    if (n >= 63) return false;
    return M < (1ull << (63 - n));
}

int bound_impl(const int64_t* data, int log2n, int64_t* scratch_dev, int dev, cudaStream_t s, uint64_t* max_abs) {
    int64_t* sc = scratch_dev;
    if (!sc) {
        void* p = nullptr;
        BW_TRY(scratch(dev, 64, &p));
        sc = reinterpret_cast<int64_t*>(p);
    }
    BW_TRY(minmax_impl(data, 1ull << log2n, sc, dev, s));
    int64_t mm[2];
    BW_CUDA(cudaMemcpyAsync(mm, sc, sizeof mm, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    const uint64_t M = magnitude(mm[0], mm[1]);
    if (max_abs) *max_abs = M;
    if (!bound_ok(M, log2n))
        return fail(BW_OVERFLOW_BOUND,
                    "max |x| = %llu with n = %d can overflow int64; need |x| * 2**n < 2**63",
                    (unsigned long long)M, log2n);
    return BW_OK;
}

}  // namespace

extern "C" {

int bw_abi_version(void) { return BW_ABI_VERSION; }

const char* bw_last_error(void) { return g_err.c_str(); }

int bw_device_cc(int device) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return major * 10 + minor;
}

// fwht_array (core.py:97-117)
int bw_fwht_i64(int64_t* data, int log2n, void* stream, uint64_t* butterflies) {
    BW_TRY(check_signal(data, log2n));
    // signals the compact plan is faster on try it first: its first pass tests
    // every input and the int64 plan takes over (after an exact restore) when
    // a value is too large for int32 intermediates; bit-identical either way
    if (compact_default(log2n, data)) return bw_fwht_i64_compact(data, log2n, -1, stream, nullptr, butterflies);
    return bw_fwht_i64_int64plan(data, log2n, stream, butterflies);
}

// fwht_array on the int64 plan, whatever the data (asynchronous; the A/B
// partner of the default above and its fallback).
int bw_fwht_i64_int64plan(int64_t* data, int log2n, void* stream, uint64_t* butterflies) {
    BW_TRY(fwht_impl(data, log2n, nullptr, false, as_stream(stream)));
    if (butterflies) *butterflies = butterfly_count(log2n);
    return BW_OK;
}

// Pass-level access to the default plan (benchmark instrumentation: one
// CUDA event per pass boundary gives each kernel's duration in the step).
int bw_plan_npasses(int log2n) {
    if (log2n < 0 || log2n > BW_MAX_LOG2N) return -fail(BW_BAD_ARGUMENTS, "log2n = %d outside 0..%d", log2n, BW_MAX_LOG2N);
    std::vector<int> w;
    default_plan(log2n, &w);
    return (int)w.size();
}

int bw_fwht_i64_pass(int64_t* data, int log2n, int pass_index, void* stream) {
    BW_TRY(check_signal(data, log2n));
    if (log2n >= bw::kCtaBits && (reinterpret_cast<uintptr_t>(data) & 15u))
        return fail(BW_BAD_ARGUMENTS, "pass-level launches need a 16-byte aligned signal");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    std::vector<int> w;
    BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    if (pass_index < 0 || pass_index >= (int)passes.size())
        return fail(BW_BAD_ARGUMENTS, "pass %d outside 0..%d", pass_index, (int)passes.size() - 1);
    return launch_pass(passes[pass_index], reinterpret_cast<u64*>(data), log2n, as_stream(stream));
}

// Pass-level launch with the threshold test fused into its epilogue (the
// benchmark's instrumented form of bw_fwht_extract_i64): hits are appended
// unordered to out_idx/out_val, their number accumulated in *count_dev.
int bw_fwht_i64_pass_extract(int64_t* data, int log2n, int pass_index, uint64_t tau, uint64_t base,
                             int64_t* out_idx, int64_t* out_val, uint64_t cap, uint64_t* count_dev, void* stream) {
    BW_TRY(check_signal(data, log2n));
    if (!count_dev || (cap > 0 && (!out_idx || !out_val))) return fail(BW_BAD_ARGUMENTS, "null extraction output");
    if (log2n >= bw::kCtaBits && (reinterpret_cast<uintptr_t>(data) & 15u))
        return fail(BW_BAD_ARGUMENTS, "pass-level launches need a 16-byte aligned signal");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    std::vector<int> w;
    BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    if (pass_index < 0 || pass_index >= (int)passes.size() || passes[pass_index].kind == SMALL)
        return fail(BW_BAD_ARGUMENTS, "pass %d cannot carry a fused extraction", pass_index);
    bw::ExtractArgs ex = {tau, base, reinterpret_cast<long long*>(out_idx), reinterpret_cast<long long*>(out_val),
                          reinterpret_cast<unsigned long long*>(count_dev), cap};
    return launch_pass(passes[pass_index], reinterpret_cast<u64*>(data), log2n, as_stream(stream), &ex);
}

// Sort up to 2048 fused-extraction hits by index in place (async).
int bw_sort_hits_i64(int64_t* idx, int64_t* val, const uint64_t* count_dev, void* stream) {
    if (!idx || !val || !count_dev) return fail(BW_BAD_ARGUMENTS, "null pointer");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    bw::k_sort_hits<<<1, 1024, 0, as_stream(stream)>>>(reinterpret_cast<long long*>(idx),
                                                       reinterpret_cast<long long*>(val),
                                                       reinterpret_cast<const unsigned long long*>(count_dev));
    BW_LAUNCHED("k_sort_hits launch");
    return BW_OK;
}

// Stages [0, sum(pass_bits)) only, on every 2^sum block of a 2^log2n array
// (the local passes of the fused multi-device plan).
int bw_fwht_i64_partial(int64_t* data, int log2n, const int* pass_bits, int npasses, void* stream) {
    BW_TRY(check_signal(data, log2n));
    if (!pass_bits || npasses < 1) return fail(BW_BAD_ARGUMENTS, "empty pass list");
    if (log2n >= bw::kCtaBits && (reinterpret_cast<uintptr_t>(data) & 15u))
        return fail(BW_BAD_ARGUMENTS, "partial transforms need a 16-byte aligned signal");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    std::vector<int> w(pass_bits, pass_bits + npasses);
    std::vector<Pass> passes;
    int covered = 0;
    for (int x : w) covered += x & 15;
    if (covered > log2n) return fail(BW_BAD_ARGUMENTS, "pass widths cover %d bits, signal has %d", covered, log2n);
    BW_TRY(build_passes(covered, w, &passes));  // the plan is validated on its own bits
    for (const Pass& p : passes) {
        if (p.kind == SMALL) return fail(BW_BAD_ARGUMENTS, "partial transforms need a 13+ bit low pass");
        BW_TRY(launch_pass(p, reinterpret_cast<u64*>(data), log2n, as_stream(stream)));
    }
    return BW_OK;
}

int bw_fwht_i64_planned(int64_t* data, int log2n, const int* pass_bits, int npasses, void* stream) {
    if (npasses < 0 || (npasses > 0 && !pass_bits)) return fail(BW_BAD_ARGUMENTS, "bad pass list");
    if (npasses == 0) return fwht_impl(data, log2n, nullptr, true, as_stream(stream));
    std::vector<int> w(pass_bits, pass_bits + npasses);
    return fwht_impl(data, log2n, &w, false, as_stream(stream));
}

// Narrow integer input, int64 output (out of place): the first pass reads
// the src_bytes-byte source (4 / 2 / 1 B per point) and writes int64, the
// rest run in place on dst -- the reference's fwht_array on
// x.astype(int64), with overflow-free int64 sums.
int bw_fwht_widen(const void* src, int src_bytes, int64_t* dst, int log2n, void* stream, uint64_t* butterflies) {
    BW_TRY(check_signal(dst, log2n));
    if (src_bytes != 1 && src_bytes != 2 && src_bytes != 4)
        return fail(BW_BAD_ARGUMENTS, "narrow sources are 1, 2 or 4 bytes per point (got %d)", src_bytes);
    if (!src || (reinterpret_cast<uintptr_t>(src) & (2u * src_bytes - 1u)))
        return fail(BW_BAD_ARGUMENTS, "narrow source must be %d-byte aligned", 2 * src_bytes);
    if (reinterpret_cast<uintptr_t>(dst) & 15u) return fail(BW_BAD_ARGUMENTS, "int64 destination must be 16-byte aligned");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    u64* d = reinterpret_cast<u64*>(dst);
    std::vector<int> w;
    BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    if (passes.empty() || passes[0].kind != LOW) {  // tiny signals: widen, then transform
        const uint64_t count = 1ull << log2n;
        const int grid = grid_for(dev, count, 256, 4);
        long long* dl = reinterpret_cast<long long*>(dst);
        if (src_bytes == 4) bw::k_widen<int><<<grid, 256, 0, s>>>(reinterpret_cast<const int*>(src), dl, count);
        else if (src_bytes == 2) bw::k_widen<short><<<grid, 256, 0, s>>>(reinterpret_cast<const short*>(src), dl, count);
        else bw::k_widen<signed char><<<grid, 256, 0, s>>>(reinterpret_cast<const signed char*>(src), dl, count);
        BW_LAUNCHED("k_widen launch");
        BW_TRY(fwht_impl(dst, log2n, nullptr, false, s));
    } else {
        BW_TRY(launch_pass(passes[0], d, log2n, s, nullptr, src, src_bytes));
        for (size_t i = 1; i < passes.size(); ++i) BW_TRY(launch_pass(passes[i], d, log2n, s));
    }
    if (butterflies) *butterflies = butterfly_count(log2n);
    return BW_OK;
}

int bw_fwht_widen_i32(const int32_t* src, int64_t* dst, int log2n, void* stream, uint64_t* butterflies) {
    return bw_fwht_widen(src, 4, dst, log2n, stream, butterflies);
}

// fwht_array on a float64 buffer (core.py:97-117): stages strictly ascending
// (2^13-element shared-memory tiles for stages 0..12, then one launch per
// stage), each stage the same IEEE a+b / a-b as numpy, so bitwise identical.
int bw_fwht_f64(double* data, int log2n, void* stream, uint64_t* butterflies) {
    BW_TRY(check_signal(data, log2n));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    BW_TRY(run_scalar_plan<true>(reinterpret_cast<u64*>(data), log2n, as_stream(stream)));
    if (butterflies) *butterflies = butterfly_count(log2n);
    return BW_OK;
}

// inverse_wht_inplace for float64 (core.py:168-169): forward then * 2^-n.
int bw_inverse_f64(double* data, int log2n, void* stream) {
    BW_TRY(bw_fwht_f64(data, log2n, stream, nullptr));
    if (log2n == 0) return BW_OK;
    int dev = 0;
    BW_TRY(device_setup(&dev));
    const uint64_t count = 1ull << log2n;
    bw::k_scale_f64<<<grid_for(dev, count, 256, 8), 256, 0, as_stream(stream)>>>(data, count, ldexp(1.0, -log2n));
    BW_LAUNCHED("k_scale_f64 launch");
    return BW_OK;
}

int bw_minmax_i64(const int64_t* data, uint64_t count, int64_t* out_minmax_dev, void* stream) {
    if (!data || !out_minmax_dev) return fail(BW_BAD_ARGUMENTS, "null pointer");
    if (count == 0) return fail(BW_BAD_ARGUMENTS, "empty signal");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    return minmax_impl(data, count, out_minmax_dev, dev, as_stream(stream));
}

// check_magnitude_bound (core.py:80-94)
int bw_check_bound_i64(const int64_t* data, int log2n, int64_t* scratch_dev, void* stream, uint64_t* max_abs) {
    BW_TRY(check_signal(data, log2n));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    return bound_impl(data, log2n, scratch_dev, dev, as_stream(stream), max_abs);
}

}  // extern "C"
namespace {
// fwht_inplace with the magnitude bound fused into the low pass (n >= 22,
// 16-byte aligned, a 13- or 14-bit first pass): the pass tests every input
// against |x| <= 2^(63-n) - 1 (core.py:80-94 element-wise) and a tile with a
// bad input writes nothing; after the pass one word says whether any tile
// failed.  Then either the other passes run (no separate 8 B/point reduction
// pass), or the tiles that did write are restored exactly -- the same stages
// again, >> w (H H = 2^w I; no wrap below the bound) -- and the call fails
// like core.py:122, before any visible mutation.  *handled = false: shape
// not covered, the caller checks the bound first.
int fused_bound_inplace(int64_t* data, int log2n, cudaStream_t s, bool* handled) {
    *handled = false;
    if (!g_fused_bound || log2n < 22 || log2n > 62 || (reinterpret_cast<uintptr_t>(data) & 15u)) return BW_OK;
    int dev = 0;
    BW_TRY(device_setup(&dev));
    std::vector<int> w;
    BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    if (passes.size() < 2 || passes[0].kind != LOW || passes[0].q > 1) return BW_OK;
    const Pass& p0 = passes[0];
    const size_t tiles = 1ull << (log2n - p0.r);
    void* sc = nullptr;
    BW_TRY(scratch(dev, 64 + 4 * tiles, &sc));
    unsigned long long* abort = reinterpret_cast<unsigned long long*>(sc);
    unsigned* flags = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(sc) + 64);
    BW_CUDA(cudaMemsetAsync(sc, 0, 64 + 4 * tiles, s));
    u64* d = reinterpret_cast<u64*>(data);
    auto low = [&](int mode, unsigned long long arg) -> int {
        return visit_pass(p0, [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            if constexpr (L >= C::T && C::Q <= 1) {
                bw::ExtractArgs ex = {};
                ex.tau = arg;
                ex.count = abort;
                ex.idx = reinterpret_cast<long long*>(flags);
                const unsigned grid = (unsigned)(1ull << (log2n - bw::kCtaBits));
                const void* none = nullptr;
                int zero = 0;
                if (mode == bw::MAP_CHECK) {
                    auto kern = bw::k_pass<C, L, false, 0, false, bw::MAP_CHECK>;
                    const int smem = bw::Dims<C>::SMEM_BYTES + (C::Q > 0 ? 8 * bw::Dims<C>::CLUSTER : 0);
                    BW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid);
                    cfg.blockDim = dim3(bw::Dims<C>::NT);
                    cfg.dynamicSmemBytes = smem;
                    cfg.stream = s;
                    cudaLaunchAttribute attr[1];
                    attr[0].id = cudaLaunchAttributeClusterDimension;
                    attr[0].val.clusterDim.x = bw::Dims<C>::CLUSTER;
                    attr[0].val.clusterDim.y = 1;
                    attr[0].val.clusterDim.z = 1;
                    cfg.attrs = attr;
                    cfg.numAttrs = C::Q > 0 ? 1 : 0;
                    BW_CUDA(cudaLaunchKernelEx(&cfg, kern, d, zero, ex, none));
                    return BW_OK;
                }
                auto kern = bw::k_pass<C, L, false, 0, false, bw::MAP_RESTORE>;
                BW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bw::Dims<C>::SMEM_BYTES));
                return launch_cfg<C>(kern, grid, s, d, zero, ex, none);
            } else {
                return fail(BW_BAD_ARGUMENTS, "no checked form of this low pass");
            }
        });
    };
    const unsigned long long lim = (1ull << (63 - log2n)) - 1ull;
    BW_TRY(low(bw::MAP_CHECK, lim));
    unsigned long long bad = 0;
    BW_CUDA(cudaMemcpyAsync(&bad, abort, sizeof bad, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    *handled = true;
    if (bad) {
        BW_TRY(low(bw::MAP_RESTORE, (unsigned long long)p0.r));
        BW_TRY(bound_impl(data, log2n, nullptr, dev, s, nullptr));  // the reference's error, with M
        return fail(BW_CUDA_ERROR, "fused bound check failed but the reduction found the bound satisfied");
    }
    for (size_t i = 1; i < passes.size(); ++i) BW_TRY(launch_pass(passes[i], d, log2n, s));
    return BW_OK;
}
}  // namespace
extern "C" {

// fwht_inplace (core.py:120-125): bound first (raise before mutation), then transform.
// Large signals check the bound inside the low pass (fused_bound_inplace);
// the others run the reduction first.  With BW_COMPACT=1 the bound M also
// picks the compact in-place plan when M <= lim(n).
int bw_fwht_inplace_i64(int64_t* data, int log2n, int64_t* scratch_dev, void* stream, uint64_t* butterflies) {
    BW_TRY(check_signal(data, log2n));
    const bool auto_compact = compact_mode() < 0 && compact_default(log2n, data);
    if (auto_compact) {
        // the compact plan's input test (|x| <= lim(n) < 2^(63-n)) is stricter
        // than the overflow bound: a signal that passes it is transformed at
        // once; otherwise the buffer is as it was and the bound is checked below
        int used = 0;
        BW_TRY(compact_try(data, log2n, as_stream(stream), &used));
        if (used) {
            if (butterflies) *butterflies = butterfly_count(log2n);
            return BW_OK;
        }
    }
    const bool g_compact = compact_mode() == 1;
    if (!g_compact) {
        bool handled = false;
        const int rc = fused_bound_inplace(data, log2n, as_stream(stream), &handled);
        if (handled) {
            if (rc == BW_OK && butterflies) *butterflies = butterfly_count(log2n);
            return rc;
        }
        if (rc != BW_OK) return rc;
    }
    uint64_t m = 0;
    BW_TRY(bw_check_bound_i64(data, log2n, scratch_dev, stream, &m));
    if (g_compact && m <= (uint64_t)0x7fffffff)
        return bw_fwht_i64_compact(data, log2n, (long long)m, stream, nullptr, butterflies);
    return bw_fwht_i64_int64plan(data, log2n, stream, butterflies);
}

// fwht_inplace with the bound M supplied by the caller (SURVEY.md 8b
// "max_abs_or_neg1"): M * 2^n < 2^63 is checked on the host, so no
// reduction pass and no stream synchronisation; max_abs < 0 falls back to
// the device check of bw_fwht_inplace_i64.
int bw_fwht_inplace_known_i64(int64_t* data, int log2n, int64_t max_abs, void* stream, uint64_t* butterflies) {
    if (max_abs < 0) return bw_fwht_inplace_i64(data, log2n, nullptr, stream, butterflies);
    BW_TRY(check_signal(data, log2n));
    if (!bound_ok(static_cast<uint64_t>(max_abs), log2n))
        return fail(BW_OVERFLOW_BOUND,
                    "max |x| = %llu with n = %d can overflow int64; need |x| * 2**n < 2**63",
                    (unsigned long long)max_abs, log2n);
    if ((compact_mode() == 1 || compact_default(log2n, data)) && max_abs <= 0x7fffffff)
        return bw_fwht_i64_compact(data, log2n, max_abs, stream, nullptr, butterflies);  // int64 plan above lim(n)
    return bw_fwht_i64_int64plan(data, log2n, stream, butterflies);
}

}  // extern "C"
namespace {
// ---- narrow intermediates (bw_fwht_i64_narrow) ----------------------------
//
// A layout is a permutation of the index bits: pos[b] = the offset bit that
// global index bit b lands on.  Natural order: pos[b] = b.  Tile-major for
// pass q: q's tile bits keep their tile-local position, q's tile-id bits
// follow above them (tiles stored one after another, in launch order).
struct Layout {
    int pos[64];
};

// Geometry of a pass: tile bits T, column bits L and the global bit of
// every virtual tile bit (one-run passes).
struct PassGeom {
    int T = 0, L = 0;
    int gb[16] = {};
    uint64_t tile_mask = 0;  // global bits that are tile bits
};

int pass_geom(const Pass& p, PassGeom* g) {
    if (p.a) return fail(BW_BAD_ARGUMENTS, "split-row passes have no narrow form");
    return visit_pass(p, [&](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        g->T = C::T;
        g->L = decltype(l)::value;
        if (g->L > g->T) g->L = g->T;
        g->tile_mask = 0;
        for (int vb = 0; vb < g->T; ++vb) {
            g->gb[vb] = vb < g->L ? vb : p.k + (vb - g->L);
            g->tile_mask |= 1ull << g->gb[vb];
        }
        return BW_OK;
    });
}

Layout natural_layout(int n) {
    Layout o;
    for (int b = 0; b < 64; ++b) o.pos[b] = b < n ? b : -1;
    return o;
}

Layout tile_major_layout(const PassGeom& q, int n) {
    Layout o;
    for (int b = 0; b < 64; ++b) o.pos[b] = -1;
    for (int vb = 0; vb < q.T; ++vb) o.pos[q.gb[vb]] = vb;
    int t = 0;
    for (int b = 0; b < n; ++b)
        if (!((q.tile_mask >> b) & 1)) o.pos[b] = q.T + t++;
    return o;
}

template <class C, int RD>
void fill_layout_tab(const PassGeom& g, int n, const Layout& lay, bw::LayoutTab* t) {
    memset(t, 0, sizeof *t);
    for (int j = 0; j < 32; ++j)
        for (int i = 0; i < C::R; ++i)
            if ((j >> i) & 1) t->reg[j] += 1ull << lay.pos[g.gb[C::reg(RD, i)]];
    for (int vb = 0; vb < g.T; ++vb) t->bit[vb] = 1ull << lay.pos[g.gb[vb]];
    // tile id bit i <-> the i-th free global bit (ascending, as tile_base enumerates)
    int tid = 0;
    for (int b = 0; b < n; ++b) {
        if ((g.tile_mask >> b) & 1) continue;
        const int d = lay.pos[b];
        const int r = t->nruns - 1;
        if (r >= 0 && t->rsrc[r] + t->rlen[r] == tid && t->rdst[r] + t->rlen[r] == d) {
            ++t->rlen[r];
        } else {
            t->rsrc[t->nruns] = tid;
            t->rlen[t->nruns] = 1;
            t->rdst[t->nruns] = d;
            ++t->nruns;
        }
        ++tid;
    }
}

enum NarrowRole { NARROW_FIRST, NARROW_MID, NARROW_LAST_FROM16, NARROW_LAST_FROM32 };

int launch_mapped(const Pass& p, int n, NarrowRole role, const void* src, void* dst, const Layout& ld,
                  const Layout& st, unsigned* flag, cudaStream_t s) {
    PassGeom g;
    BW_TRY(pass_geom(p, &g));
    return visit_pass(p, [&](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        constexpr int L = decltype(l)::value;
        if constexpr (C::Q > 1 || bw::SplitOf<C>::value) {
            return fail(BW_BAD_ARGUMENTS, "no narrow form of this pass shape");
        } else {
            bw::MapArgs m;
            fill_layout_tab<C, 0>(g, n, ld, &m.ld);
            fill_layout_tab<C, C::NR - 1>(g, n, st, &m.st);
            if (m.ld.nruns > 6 || m.st.nruns > 6) return fail(BW_BAD_ARGUMENTS, "layout needs too many runs");
            m.lim = 32767;
            const unsigned grid = (unsigned)(1ull << (n - bw::kCtaBits));
            constexpr int smem = bw::Dims<C>::SMEM_BYTES;
            constexpr bool kLow = L >= C::T;
            auto go = [&](auto kern, const auto* sp, auto* dp) -> int {
                if (smem > 48 * 1024) BW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                return launch_cfg<C>(kern, grid, s, sp, dp, flag, m);
            };

            if constexpr (kLow) {
                if (role != NARROW_FIRST) return fail(BW_BAD_ARGUMENTS, "a low pass is only the first narrow pass");
                return go(bw::k_pass_map<C, L, long long, short>, reinterpret_cast<const long long*>(src),
                          reinterpret_cast<short*>(dst));
            } else {
                // narrow sources: TPC tiles per CTA / cluster (BW_NARROW_TPC, experiment knob)
                auto go_tpc = [&](auto k1, auto k2, auto k4, const auto* sp, auto* dp) -> int {
                    if constexpr (C::Q <= 1) {
                        if (g_narrow_tpc == 2) {
                            if (smem > 48 * 1024) BW_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                            return launch_cfg<C>(k2, grid / 2, s, sp, dp, flag, m);
                        }
                        if (g_narrow_tpc == 4) {
                            if (smem > 48 * 1024) BW_CUDA(cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                            return launch_cfg<C>(k4, grid / 4, s, sp, dp, flag, m);
                        }
                    }
                    return go(k1, sp, dp);
                };
                constexpr int T2 = C::Q <= 1 ? 2 : 1, T4 = C::Q <= 1 ? 4 : 1;
                if (role == NARROW_MID)
                    return go_tpc(bw::k_pass_map<C, L, short, int>, bw::k_pass_map<C, L, short, int, T2>,
                                  bw::k_pass_map<C, L, short, int, T4>, reinterpret_cast<const short*>(src),
                                  reinterpret_cast<int*>(dst));
                if (role == NARROW_LAST_FROM16)
                    return go_tpc(bw::k_pass_map<C, L, short, long long>, bw::k_pass_map<C, L, short, long long, T2>,
                                  bw::k_pass_map<C, L, short, long long, T4>, reinterpret_cast<const short*>(src),
                                  reinterpret_cast<long long*>(dst));
                if (role == NARROW_LAST_FROM32)
                    return go_tpc(bw::k_pass_map<C, L, int, long long>, bw::k_pass_map<C, L, int, long long, T2>,
                                  bw::k_pass_map<C, L, int, long long, T4>, reinterpret_cast<const int*>(src),
                                  reinterpret_cast<long long*>(dst));
                return fail(BW_BAD_ARGUMENTS, "a high pass is never the first narrow pass");
            }
        }
    });
}

// Plans with a narrow form: a low pass of 13 or 14 bits, then one or two
// one-run high passes on tiles of one or two CTAs.
bool narrow_plan(int n, std::vector<Pass>* passes) {
    std::vector<int> w;
    if (default_plan(n, &w, true) != BW_OK) return false;
    if (build_passes(n, w, passes) != BW_OK) return false;
    if (passes->size() < 2 || passes->size() > 3 || (*passes)[0].kind != LOW || (*passes)[0].q > 1) return false;
    for (size_t i = 1; i < passes->size(); ++i)
        if ((*passes)[i].a || (*passes)[i].q > 1 || (*passes)[i].r > 16) return false;
    return true;
}

uint64_t narrow_scratch_bytes(int n, size_t npasses) {
    return (2ull << n) + (npasses == 3 ? (4ull << n) : 0ull);
}

// Pass i of the narrow plan: 0 = int64 -> int16 (flags values over
// +-32767), then int16 -> int32 -> int64 (three passes) or int16 -> int64.
int narrow_pass(int64_t* data, int n, void* work, const std::vector<Pass>& passes, int i, unsigned* flag,
                cudaStream_t s) {
    std::vector<PassGeom> g(passes.size());
    for (size_t q = 0; q < passes.size(); ++q) BW_TRY(pass_geom(passes[q], &g[q]));
    short* a16 = reinterpret_cast<short*>(work);
    int* b32 = reinterpret_cast<int*>(reinterpret_cast<char*>(work) + (2ull << n));
    const Layout nat = natural_layout(n);
    const Layout tm1 = tile_major_layout(g[1], n);
    if (i == 0) return launch_mapped(passes[0], n, NARROW_FIRST, data, a16, nat, tm1, flag, s);
    if (passes.size() == 2) return launch_mapped(passes[1], n, NARROW_LAST_FROM16, a16, data, tm1, nat, flag, s);
    const Layout tm2 = tile_major_layout(g[2], n);
    if (i == 1) return launch_mapped(passes[1], n, NARROW_MID, a16, b32, tm1, tm2, flag, s);
    return launch_mapped(passes[2], n, NARROW_LAST_FROM32, b32, data, tm2, nat, flag, s);
}

int narrow_args(int64_t* data, int log2n, void* work, uint64_t work_bytes, std::vector<Pass>* passes) {
    BW_TRY(check_signal(data, log2n));
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !narrow_plan(log2n, passes))
        return fail(BW_BAD_ARGUMENTS, "no narrow plan for this signal (n = %d)", log2n);
    const uint64_t need = narrow_scratch_bytes(log2n, passes->size());
    if (!work || work_bytes < need || (reinterpret_cast<uintptr_t>(work) & 15u))
        return fail(BW_BAD_ARGUMENTS, "narrow work buffer needs %llu bytes, 16-byte aligned (bw_narrow_scratch_bytes)",
                    (unsigned long long)need);
    return BW_OK;
}
}  // namespace
extern "C" {

uint64_t bw_narrow_scratch_bytes(int log2n) {
    if (log2n < 0 || log2n > BW_MAX_LOG2N) return 0;
    std::vector<Pass> passes;
    if (!narrow_plan(log2n, &passes)) return 0;
    return narrow_scratch_bytes(log2n, passes.size());
}

int bw_narrow_npasses(int log2n) {
    std::vector<Pass> passes;
    if (log2n < 0 || log2n > BW_MAX_LOG2N || !narrow_plan(log2n, &passes)) return 0;
    return (int)passes.size();
}

// One pass of the narrow plan, asynchronous (benchmark instrumentation and
// callers that check the flag themselves): pass 0 ORs 1 into *flag_dev when
// a value does not fit int16 -- the signal is then untouched and the caller
// must run the int64 plan instead of the later passes.
int bw_fwht_i64_narrow_pass(int64_t* data, int log2n, void* work, uint64_t work_bytes, int pass_index,
                            uint32_t* flag_dev, void* stream) {
    std::vector<Pass> passes;
    BW_TRY(narrow_args(data, log2n, work, work_bytes, &passes));
    if (pass_index < 0 || pass_index >= (int)passes.size() || (pass_index == 0 && !flag_dev))
        return fail(BW_BAD_ARGUMENTS, "bad narrow pass %d (or null flag)", pass_index);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    return narrow_pass(data, log2n, work, passes, pass_index, reinterpret_cast<unsigned*>(flag_dev), as_stream(stream));
}

// Static checker of the narrow plan (TEST HOOK, n <= 24): runs the mapped
// kernels' exact address computation (layout tables, thread / rank parts,
// tile runs) for every element of every pass and checks that pass 0 loads
// and the last pass stores in natural order, that every store offset is a
// bijection onto [0, 2^n), and that pass i+1 loads every element exactly
// where pass i stored it.
int bw_plan_check_narrow(int log2n) {
    if (log2n < 16 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "narrow plan check supports 16 <= n <= 24");
    std::vector<Pass> passes;
    if (!narrow_plan(log2n, &passes)) return fail(BW_BAD_ARGUMENTS, "no narrow plan for n = %d", log2n);
    const uint64_t N = 1ull << log2n;
    std::vector<PassGeom> g(passes.size());
    for (size_t q = 0; q < passes.size(); ++q) BW_TRY(pass_geom(passes[q], &g[q]));
    std::vector<Layout> lay;  // layout between pass q-1 and pass q (lay[0] = input)
    lay.push_back(natural_layout(log2n));
    for (size_t q = 1; q < passes.size(); ++q) lay.push_back(tile_major_layout(g[q], log2n));
    lay.push_back(natural_layout(log2n));
    std::vector<uint64_t> ld(N), st(N);
    std::vector<uint8_t> seen(N);
    auto base_of = [](const bw::LayoutTab& t, uint64_t tile, uint32_t vt) {
        unsigned long long off = 0;
        for (int r = 0; r < t.nruns; ++r) off += ((tile >> t.rsrc[r]) & ((1ull << t.rlen[r]) - 1ull)) << t.rdst[r];
        for (int b = 0; b < 16; ++b)
            if ((vt >> b) & 1u) off += t.bit[b];
        return off;
    };
    std::vector<uint64_t> prev_st;
    for (size_t q = 0; q < passes.size(); ++q) {
        const int st_ok = visit_pass(passes[q], [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            constexpr int T = C::T, NQ = 1 << C::Q, LAST = C::NR - 1;
            if constexpr (C::Q > 1 || bw::SplitOf<C>::value) {
                return fail(BW_BAD_ARGUMENTS, "no narrow form");
            } else {
                bw::LayoutTab tl, ts;
                fill_layout_tab<C, 0>(g[q], log2n, lay[q], &tl);
                fill_layout_tab<C, LAST>(g[q], log2n, lay[q + 1], &ts);
                std::fill(seen.begin(), seen.end(), 0);
                const uint64_t ctas = 1ull << (log2n - bw::kCtaBits);
                for (uint64_t cta = 0; cta < ctas; ++cta) {
                    const uint32_t rank = (uint32_t)(cta & (NQ - 1));
                    const uint64_t tile = cta >> C::Q;
                    const uint64_t gbase = bw::tile_base<T, L>(tile, passes[q].k);
                    for (uint32_t th = 0; th < (uint32_t)bw::Dims<C>::NT; ++th) {
                        const uint32_t lane = th & 31u, warp = th >> 5;
                        const uint32_t v0 = bw::thread_part<C, 0>(lane, warp) | bw::rank_bits<C, 0>(rank);
                        const uint32_t v1 = bw::thread_part<C, LAST>(lane, warp) | bw::rank_bits<C, LAST>(rank);
                        const uint64_t b0 = base_of(tl, tile, v0), b1 = base_of(ts, tile, v1);
                        for (int j = 0; j < bw::Dims<C>::E; ++j) {
                            const uint64_t gi = gbase + bw::global_off<T, L>(v0 | bw::reg_part<C, 0>(j), passes[q].k);
                            const uint64_t go = gbase + bw::global_off<T, L>(v1 | bw::reg_part<C, LAST>(j), passes[q].k);
                            if (gi >= N || go >= N) return fail(BW_BAD_ARGUMENTS, "pass %d leaves the signal", (int)q);
                            ld[gi] = b0 + tl.reg[j];
                            st[go] = b1 + ts.reg[j];
                            if (st[go] >= N || seen[st[go]]) return fail(BW_BAD_ARGUMENTS, "pass %d stores twice", (int)q);
                            seen[st[go]] = 1;
                        }
                    }
                }
                return BW_OK;
            }
        });
        if (st_ok != BW_OK) return st_ok;
        for (uint64_t i = 0; i < N; ++i) {
            if (q == 0 && ld[i] != i) return fail(BW_BAD_ARGUMENTS, "pass 0 does not load in natural order");
            if (q > 0 && ld[i] != prev_st[i]) return fail(BW_BAD_ARGUMENTS, "pass %d loads index %llu elsewhere", (int)q,
                                                          (unsigned long long)i);
            if (q + 1 == passes.size() && st[i] != i) return fail(BW_BAD_ARGUMENTS, "last pass does not store in natural order");
        }
        prev_st = st;
    }
    return BW_OK;
}

// fwht_array with narrow intermediates: pass 1 reads int64 and writes int16
// (checked: every value after the low pass within +-32767), a middle pass
// writes int32 (exact: |y| <= 32767 * 2^r < 2^31 for r <= 16), the last
// pass writes int64 back in place; each intermediate is stored tile-major
// for the pass that reads it.  When a value does not fit, the signal is
// still untouched (pass 1 only read it) and the int64 plan runs instead.
// Synchronises the stream once (the overflow flag after pass 1).  Plans
// without a narrow form (n < 16, split rows, 4-CTA tiles) run the int64 plan.
int bw_fwht_i64_narrow(int64_t* data, int log2n, void* work, uint64_t work_bytes, void* stream,
                       int* used_narrow, uint64_t* butterflies) {
    BW_TRY(check_signal(data, log2n));
    if (used_narrow) *used_narrow = 0;
    if (butterflies) *butterflies = butterfly_count(log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    std::vector<Pass> passes;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !narrow_plan(log2n, &passes))
        return fwht_impl(data, log2n, nullptr, false, s);
    BW_TRY(narrow_args(data, log2n, work, work_bytes, &passes));
    void* sc = nullptr;
    BW_TRY(scratch(dev, 64, &sc));
    unsigned* flag = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(sc) + 40);
    BW_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned), s));
    BW_TRY(narrow_pass(data, log2n, work, passes, 0, flag, s));
    unsigned bad = 0;
    BW_CUDA(cudaMemcpyAsync(&bad, flag, sizeof bad, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (bad) return fwht_impl(data, log2n, nullptr, false, s);  // data untouched: the int64 plan
    for (size_t i = 1; i < passes.size(); ++i) BW_TRY(narrow_pass(data, log2n, work, passes, (int)i, flag, s));
    if (used_narrow) *used_narrow = 1;
    return BW_OK;
}

}  // extern "C"
namespace {
// ---- compact in-place intermediates (bw_fwht_i64_compact) -----------------
//
// For signals with small values (the +-1 Boolean signals of the paper, any
// |x| <= lim(n)) every pass but the last can keep the signal as int32, and
// the signal's own buffer holds the int32 copy: no work buffer.  Stages
// commute (Z/2^64), so the plan runs its HIGH passes first, in int32, and the
// low pass last, which widens to int64 and writes the natural order:
//   P1: natural int64 -> int32,  P2..Pm: int32 -> int32,  C: int32 -> int64
// = 12 + 8*(m-1) + 12 bytes per point instead of 16 * (m+1).
//
// Layouts.  w = the low pass's width (13 or 14 bits), c = w - 1.  A "block"
// is the 2^w contiguous int64 slots of one low-pass tile = 2^(w+1) int32
// slots; its half h holds the int32 copy of the block's 2^w elements:
//   int32 slot = block << (w+1) | h << w | perm(i mod 2^w),
//   perm: i0..i3 -> slot bits 0..3, i_c -> bit 4, i4..i_(c-1) -> bits 5..c.
// Every high pass's tile contains the bits {0,1,2,3,c} (plus low bits 4, 5,
// .. when it has fewer than 9 stage rows) as its non-stage "columns", so a
// 128-byte int32 segment is 32 elements of ONE tile for every pass.
// In-place safety (bw_plan_check_compact proves it on the exact tables):
//   P1 reads every int64 slot; tile t's outputs land in its own rows with
//     i_c = h (it contains bit c), i.e. inside what t itself read.
//   P_j (j >= 2) reads half h_(j-1) and writes the other half, which no tile
//     reads in that pass.
//   C reads the half of its own block and writes the whole block.
// lim(n) = (2^31 - 1) >> (n - w): no int32 value of the high passes wraps.
// Unknown magnitudes: P1 tests every input; a tile with |x| > lim (or one
// that starts after another failed) writes nothing and every CTA of its
// cluster agrees; written tiles are marked.  After a failure the marked
// tiles are restored exactly -- P1's stages again on their int32 copy, then
// >> r1 (H H = 2^r1 I) -- and the int64 plan runs.
struct CompactPlan {
    int n = 0, w = 0, c = 0, m = 0;  // m high passes, then the low pass
    bool v2 = false;                  // passes after the first on the int32 engine (bw_kernels32.cuh)
    bool first32 = false;             // v2 and the first pass on it too (8 or 9 rows)
    std::vector<Pass> pass;           // shapes for the kernel visitor
    std::vector<PassGeom> geom;
    std::vector<int> half;            // half written by high pass j
    long long lim = 0;
};

// BW_COMPACT_ROWS="r1,r2,..": stage rows of the high passes (experiments;
// default: balanced, at most 9).  BW_COMPACT_W=13|14: the low pass width.
//
// v2 (n <= 32, the default; BW_COMPACT_V2=0 selects v1): the passes after
// the first run on the int32 engine -- k32_high (8 or 9 rows, 2^14 int32 per
// CTA) and the 14-bit low pass k32_low, whose last four stages (bits 10..13)
// run in int64 registers.  So v2 admits |x| <= (2^31 - 1) >> (n - 4): every
// stage but the last four keeps |value| <= 2^31 - 1.  Rows: one high pass
// for H <= 9; H = 10..13: H - 8 then 8; H = 14..16: 8 then H - 8 (k32_high of
// 6, 7 or 8 rows); H = 17, 18: 9 then 8 / 9 (BW_COMPACT_R2=6..9 forces the
// second pass's rows).  A FIRST pass of 8 or 9 rows also runs on
// the int32 engine (k32_first: natural int64 -> int32, the input test of the
// unknown-bound case inside it; BW_COMPACT_FIRST=0: the int64 engine's
// k_pass_map as before).
bool compact_v2_enabled() { return !(getenv("BW_COMPACT_V2") && getenv("BW_COMPACT_V2")[0] == '0'); }
bool compact_first32_enabled() { return !(getenv("BW_COMPACT_FIRST") && getenv("BW_COMPACT_FIRST")[0] == '0'); }

bool compact_plan(int n, CompactPlan* cp) {
    if (n < 16 || n > 36) return false;
    std::vector<int> rows;
    int sum = 0;
    const char* rows_env = getenv("BW_COMPACT_ROWS");
    for (const char* q = rows_env; q && *q;) {
        const int r = atoi(q);
        rows.push_back(r);
        sum += r;
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
    }
    // v2 unless disabled, n > 32, a low-pass width is forced, or forced rows
    // do not fit the int32 engine (one high pass, or a second of 8 / 9 rows)
    bool v2 = compact_v2_enabled() && n <= 35 && !getenv("BW_COMPACT_W");
    if (v2 && rows_env)
    {   // ... a first pass of any shape, later ones of 6..9 (k32_high) or 1..4 rows (k32_reg)
        bool ok = sum == n - 14 && !rows.empty() && rows.size() <= 3;
        for (size_t j = 1; ok && j < rows.size(); ++j) ok = rows[j] >= 1 && rows[j] <= 9 && rows[j] != 5;
        v2 = ok;
    }
    int w = n <= 31 ? 13 : 14;
    if (const char* e = getenv("BW_COMPACT_W")) w = atoi(e) == 14 ? 14 : 13;
    if (v2) w = 14;
    const int H = n - w;
    if (rows_env) {
        if (sum != H) return false;
    } else if (v2) {
        // H < 14: a short first pass (registers only on the int64 engine, fast) then 8 rows; H = 14..16: 8 rows
        // on the int32 engine first (256-byte segments), then H - 8 = 6..8; H = 17, 18: 9 then 8 / 9
        int r2 = H < 14 ? 8 : H <= 16 ? H - 8 : H - 9;
        if (const char* e = getenv("BW_COMPACT_R2")) r2 = atoi(e) >= 6 && atoi(e) <= 9 ? atoi(e) : 9;
        if (H <= 9) rows.push_back(H);
        else if (H >= 19 && H <= 21 && !getenv("BW_COMPACT_R2")) {  // n = 33..35: 9 rows, 8 rows, then 2..4 in registers
            rows.push_back(9);
            rows.push_back(8);
            rows.push_back(H - 17);
        } else if (H - r2 >= 1 && H - r2 <= 9) {
            rows.push_back(H - r2);
            rows.push_back(r2);
        } else return false;
    } else {
        const int m = (H + 8) / 9;
        for (int j = 0; j < m; ++j) rows.push_back(H / m + (j < H % m ? 1 : 0));
    }
    if (rows.empty() || rows.size() > 4) return false;
    cp->n = n;
    cp->w = w;
    cp->c = w - 1;
    cp->m = (int)rows.size();
    cp->v2 = v2;
    cp->first32 = v2 && compact_first32_enabled() && (rows[0] == 8 || rows[0] == 9);
    cp->lim = 0x7fffffffll >> (v2 ? n - 4 : H);
    cp->pass.clear();
    cp->geom.clear();
    cp->half.clear();
    int k = w;
    for (int j = 0; j < cp->m; ++j) {
        const int r = rows[j];
        if (r < 1 || r > 9) return false;
        Pass p;
        p.kind = r <= 5 ? REG : HIGH;
        p.q = r <= 5 ? 0 : 1;
        p.k = k;
        p.r = r;
        const int T = r <= 5 ? bw::CfgReg::T : bw::CfgHigh14c::T;
        PassGeom g;
        g.T = T;
        g.L = T - r;
        int vb = 0;
        for (int b = 0; b < 4; ++b) g.gb[vb++] = b;
        g.gb[vb++] = cp->c;
        for (int b = 4; vb < g.L; ++b) g.gb[vb++] = b;  // extra columns: low bits 4, 5, .. (all < c)
        for (int i = 0; i < r; ++i) g.gb[vb++] = k + i;
        g.tile_mask = 0;
        for (int i = 0; i < T; ++i) g.tile_mask |= 1ull << g.gb[i];
        cp->pass.push_back(p);
        cp->geom.push_back(g);
        cp->half.push_back((cp->m - 1 - j) & 1);  // the last high pass writes half 0
        k += r;
    }
    Pass low;
    low.kind = LOW;
    low.q = w == 14 ? 1 : 0;
    low.k = 0;
    low.r = w;
    PassGeom g;
    g.T = w;
    g.L = w;
    for (int b = 0; b < w; ++b) g.gb[b] = b;
    g.tile_mask = (1ull << w) - 1ull;
    cp->pass.push_back(low);
    cp->geom.push_back(g);
    return true;
}

// int32 layout of the half-block copies (offset bit of every index bit; the
// half h is the pointer offset h << w).
Layout compact_layout(const CompactPlan& cp) {
    Layout o;
    for (int b = 0; b < 64; ++b) o.pos[b] = -1;
    for (int b = 0; b < 4; ++b) o.pos[b] = b;
    o.pos[cp.c] = 4;
    for (int b = 4; b < cp.c; ++b) o.pos[b] = b + 1;
    for (int b = cp.w; b < cp.n; ++b) o.pos[b] = b + 1;
    if (getenv("BW_COMPACT_BREAK")) {  // test hook: NOT in place (bit c trades places with the top bit)
        const int t = o.pos[cp.c];
        o.pos[cp.c] = o.pos[cp.n - 1];
        o.pos[cp.n - 1] = t;
    }
    return o;
}

template <class F>
int visit_compact(const Pass& p, F&& f) {
    if (p.kind == LOW) {
        if (p.q == 0) return f(tag<bw::CfgLow13>{}, ic<13>{});
        return f(tag<bw::CfgLow14c>{}, ic<14>{});
    }
    if (p.kind == REG) return with_L<bw::CfgReg, 8, 12>(bw::CfgReg::T - p.r, f);
    if (p.kind == HIGH && p.q == 1) return with_L<bw::CfgHigh14c, 5, 8>(bw::CfgHigh14c::T - p.r, f);
    return fail(BW_BAD_ARGUMENTS, "no compact form of this pass shape");
}

enum CompactMode { COMPACT_PLAIN, COMPACT_CHECK, COMPACT_RESTORE };

// Pass i of the compact plan (i < m: high pass i; i == m: the low pass).
// mode CHECK / RESTORE apply to pass 0 only.
// ex (the low pass on the int32 engine only): the fused threshold extraction.
int launch_compact(const CompactPlan& cp, int i, int64_t* data, CompactMode mode, unsigned* tileflag,
                   unsigned* abort, cudaStream_t s, const bw::ExtractArgs* ex = nullptr) {
    const Layout nat = natural_layout(cp.n), lam = compact_layout(cp);
    int* d32 = reinterpret_cast<int*>(data);
    long long* d64 = reinterpret_cast<long long*>(data);
    const Pass& p = cp.pass[i];
    const PassGeom& g = cp.geom[i];
    const int tpc = getenv("BW_COMPACT_TPC") ? atoi(getenv("BW_COMPACT_TPC")) : 1;
    if (cp.v2 && (i > 0 || cp.first32)) {  // the int32 engine: 2^14 elements per CTA, no cluster
        const unsigned grid = (unsigned)(1ull << (cp.n - bw::w32::kBits));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(bw::w32::kNT);
        cfg.dynamicSmemBytes = bw::w32::kSmemBytes;
        cfg.stream = s;
        if (i == 0) {  // natural int64 -> int32 (plain / input test), or the restore of the tiles it wrote
            namespace w = bw::w32;
            const unsigned long long* s64 = reinterpret_cast<const unsigned long long*>(data);
            unsigned long long* d64u = reinterpret_cast<unsigned long long*>(data);
            uint32_t* h32 = reinterpret_cast<uint32_t*>(d32 + ((size_t)cp.half[0] << cp.w));
            const uint32_t lim = (uint32_t)cp.lim;
            if (mode != COMPACT_PLAIN && !tileflag) return fail(BW_BAD_ARGUMENTS, "checked / restore passes need tile flags");
            if (mode == COMPACT_CHECK && !abort) return fail(BW_BAD_ARGUMENTS, "a checked pass needs the abort word");
            if (p.r == 9) {
                if (mode == COMPACT_RESTORE) BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_restore<5>, (const uint32_t*)h32, d64u, p.k, (const unsigned*)tileflag));
                else if (mode == COMPACT_CHECK) BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_first<5, w::FIRST_CHECK>, s64, h32, p.k, lim, tileflag, abort));
                else BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_first<5, w::FIRST_PLAIN>, s64, h32, p.k, lim, (unsigned*)nullptr, (unsigned*)nullptr));
            } else {
                if (mode == COMPACT_RESTORE) BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_restore<6>, (const uint32_t*)h32, d64u, p.k, (const unsigned*)tileflag));
                else if (mode == COMPACT_CHECK) BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_first<6, w::FIRST_CHECK>, s64, h32, p.k, lim, tileflag, abort));
                else BW_CUDA(cudaLaunchKernelEx(&cfg, w::k32_first<6, w::FIRST_PLAIN>, s64, h32, p.k, lim, (unsigned*)nullptr, (unsigned*)nullptr));
            }
            return BW_OK;
        }
        const uint32_t* src = reinterpret_cast<const uint32_t*>(d32 + ((size_t)cp.half[i - 1] << cp.w));
        if (i == cp.m) {
            unsigned long long* d64u = reinterpret_cast<unsigned long long*>(data);
            if (ex) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_low<true>, src, d64u, *ex));
            else BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_low<false>, src, d64u, bw::ExtractArgs{}));
            return BW_OK;
        }
        if (ex) return fail(BW_BAD_ARGUMENTS, "only the compact plan's low pass carries the extraction");
        uint32_t* dst = reinterpret_cast<uint32_t*>(d32 + ((size_t)cp.half[i] << cp.w));
        if (p.r == 9) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_high<5>, src, dst, p.k));
        else if (p.r == 8) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_high<6>, src, dst, p.k));
        else if (p.r == 7) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_high<7>, src, dst, p.k));
        else if (p.r == 6) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_high<8>, src, dst, p.k));
        else if (p.r >= 1 && p.r <= 4) {  // registers only: 4 slots of every row per thread
            cfg.gridDim = dim3((unsigned)(1ull << (cp.n - p.r - 10)));
            cfg.dynamicSmemBytes = 0;
            if (p.r == 1) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_reg<1>, src, dst, p.k));
            else if (p.r == 2) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_reg<2>, src, dst, p.k));
            else if (p.r == 3) BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_reg<3>, src, dst, p.k));
            else BW_CUDA(cudaLaunchKernelEx(&cfg, bw::w32::k32_reg<4>, src, dst, p.k));
        }
        else return fail(BW_BAD_ARGUMENTS, "no int32-engine pass of %d rows", p.r);
        return BW_OK;
    }
    if (ex) return fail(BW_BAD_ARGUMENTS, "the fused extraction needs the int32 engine's low pass");
    return visit_compact(p, [&](auto t, auto l) -> int {
        using C = typename decltype(t)::type;
        constexpr int L = decltype(l)::value;
        constexpr bool kLow = L >= C::T;
        bw::MapArgs m;
        memset(&m, 0, sizeof m);
        m.tileflag = tileflag;
        m.abort = abort;
        m.lim = cp.lim;
        const unsigned grid = (unsigned)(1ull << (cp.n - bw::kCtaBits));
        constexpr int smem = bw::Dims<C>::SMEM_BYTES;
        auto go = [&](auto kern, unsigned gr, int sm_bytes, const auto* sp, auto* dp) -> int {
            if (sm_bytes > 48 * 1024)
                BW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_bytes));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(gr);
            cfg.blockDim = dim3(bw::Dims<C>::NT);
            cfg.dynamicSmemBytes = sm_bytes;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = bw::Dims<C>::CLUSTER;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = C::Q > 0 ? 1 : 0;
            BW_CUDA(cudaLaunchKernelEx(&cfg, kern, sp, dp, (unsigned*)nullptr, m));
            return BW_OK;
        };
        if constexpr (kLow) {
            if (i != cp.m) return fail(BW_BAD_ARGUMENTS, "the low pass is the compact plan's last");
            fill_layout_tab<C, 0>(g, cp.n, lam, &m.ld);
            fill_layout_tab<C, C::NR - 1>(g, cp.n, nat, &m.st);
            if (m.ld.nruns > 6 || m.st.nruns > 6) return fail(BW_BAD_ARGUMENTS, "layout needs too many runs");
            return go(bw::k_pass_map<C, L, int, long long>, grid, smem, d32 + ((size_t)cp.half[cp.m - 1] << cp.w), d64);
        } else {
            if (i >= cp.m) return fail(BW_BAD_ARGUMENTS, "bad compact pass %d", i);
            int* dst32 = d32 + ((size_t)cp.half[i] << cp.w);
            if (i == 0) {
                if (mode == COMPACT_RESTORE) {  // the int32 copy -> P1's stages again -> >> r -> natural int64
                    fill_layout_tab<C, 0>(g, cp.n, lam, &m.ld);
                    fill_layout_tab<C, C::NR - 1>(g, cp.n, nat, &m.st);
                    m.shift = p.r;
                    return go(bw::k_pass_map<C, L, int, long long, 1, bw::MAP_RESTORE>, grid, smem, dst32, d64);
                }
                fill_layout_tab<C, 0>(g, cp.n, nat, &m.ld);
                fill_layout_tab<C, C::NR - 1>(g, cp.n, lam, &m.st);
                if (mode == COMPACT_CHECK)
                    return go(bw::k_pass_map<C, L, long long, int, 1, bw::MAP_CHECK>, grid,
                              smem + (C::Q > 0 ? 8 * bw::Dims<C>::CLUSTER : 0), d64, dst32);
                return go(bw::k_pass_map<C, L, long long, int>, grid, smem, d64, dst32);
            }
            fill_layout_tab<C, 0>(g, cp.n, lam, &m.ld);
            fill_layout_tab<C, C::NR - 1>(g, cp.n, lam, &m.st);
            const int* src32 = d32 + ((size_t)cp.half[i - 1] << cp.w);
            if constexpr (C::Q <= 1) {
                if (tpc == 2) return go(bw::k_pass_map<C, L, int, int, 2>, grid / 2, smem, src32, dst32);
            }
            return go(bw::k_pass_map<C, L, int, int>, grid, smem, src32, dst32);
        }
    });
}

int compact_scratch(int dev, const CompactPlan& cp, unsigned** tileflag, unsigned** abort, cudaStream_t s) {
    const size_t tiles = 1ull << (cp.n - cp.geom[0].T);
    void* sc = nullptr;
    BW_TRY(scratch(dev, 64 + 4 * tiles, &sc));
    *abort = reinterpret_cast<unsigned*>(sc);
    *tileflag = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(sc) + 64);
    BW_CUDA(cudaMemsetAsync(sc, 0, 64 + 4 * tiles, s));
    return BW_OK;
}

// The compact plan on a signal of unknown magnitude: the first pass tests
// every input (one stream synchronisation to read the verdict).  *used = 1:
// the transform is done (asynchronously).  *used = 0: an input was too large
// (or there is no plan): the buffer holds the caller's input again.
// ex: the threshold extraction fused into the low pass (v2 plans only).
int compact_try(int64_t* data, int log2n, cudaStream_t s, int* used, const bw::ExtractArgs* ex) {
    *used = 0;
    CompactPlan cp;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !compact_plan(log2n, &cp) || (ex && !cp.v2)) return BW_OK;
    // the verdict readback synchronises the stream, which a capturing stream cannot do: the int64 plan then
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return BW_OK;
    }
    int dev = 0;
    BW_TRY(device_setup(&dev));
    unsigned *tileflag = nullptr, *abort = nullptr;
    BW_TRY(compact_scratch(dev, cp, &tileflag, &abort, s));
    unsigned bad = 0;
    if (cp.v2 && log2n >= 33) {  // a sample first: a refused full attempt would cost ~2.5 ms at n = 34
        bw::w32::k32_sample<<<1, bw::w32::kNT, 0, s>>>(reinterpret_cast<const unsigned long long*>(data), (uint32_t)cp.lim,
                                                        abort);
        BW_LAUNCHED("k32_sample launch");
        BW_CUDA(cudaMemcpyAsync(&bad, abort, sizeof bad, cudaMemcpyDeviceToHost, s));
        BW_CUDA(cudaStreamSynchronize(s));
        if (bad) return BW_OK;  // nothing was written
    }
    BW_TRY(launch_compact(cp, 0, data, COMPACT_CHECK, tileflag, abort, s));
    BW_CUDA(cudaMemcpyAsync(&bad, abort, sizeof bad, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (bad) return launch_compact(cp, 0, data, COMPACT_RESTORE, tileflag, abort, s);
    for (int i = 1; i <= cp.m; ++i)
        BW_TRY(launch_compact(cp, i, data, COMPACT_PLAIN, nullptr, nullptr, s, i == cp.m ? ex : nullptr));
    *used = 1;
    return BW_OK;
}

// Whether fwht_array / fwht_inplace try the compact plan on this signal
// without being asked (BW_COMPACT, see compact_mode): in auto mode the sizes
// where the checked plan, its verdict readback included, measured faster
// than the int64 plan on +-1 signals (profiles/r02_compact/passes.log):
// n = 32: 23.7 vs 31.4 ms, 31: 11.3 vs 15.5, 30: 5.57 vs 7.72, 29: 3.22 vs
// 3.88, 28: 1.63 vs 1.93, 27: 0.69 vs 0.97, 26: 0.36 vs 0.49 (n = 25: 0.197
// vs 0.224, n = 24: 0.115 vs 0.107 -- left to the int64 plan, which stays
// asynchronous).  n = 33 / 34 (lim = 3 / 1: +-1 signals): 52.0 vs 66.2 and
// 103.7 vs 141.3 ms (profiles/r02_compact/passes_n33_n34.log).
constexpr int kCompactAutoMin = 26;
constexpr int kCompactAutoMax = 34;  // n = 33, 34: three high passes (the third in registers); lim(n) = 3, 1
bool compact_default(int log2n, const void* data) {
    const int mode = compact_mode();
    if (mode == 0 || (reinterpret_cast<uintptr_t>(data) & 15u)) return false;
    CompactPlan cp;
    if (log2n < 22 || !compact_plan(log2n, &cp)) return false;
    return mode == 1 || (cp.v2 && log2n >= kCompactAutoMin && log2n <= kCompactAutoMax);
}
}  // namespace
extern "C" {

// Whether bw_fwht_i64 / bw_fwht_inplace_i64 try the compact plan on a
// 16-byte aligned signal of this size (BW_COMPACT and the measured range).
int bw_compact_auto(int log2n) { return log2n >= 0 && log2n <= BW_MAX_LOG2N && compact_default(log2n, nullptr) ? 1 : 0; }

long long bw_compact_limit(int log2n) {
    CompactPlan cp;
    if (log2n < 0 || log2n > BW_MAX_LOG2N || !compact_plan(log2n, &cp)) return -1;
    return cp.lim;
}

int bw_compact_npasses(int log2n) {
    CompactPlan cp;
    if (log2n < 0 || log2n > BW_MAX_LOG2N || !compact_plan(log2n, &cp)) return 0;
    return cp.m + 1;
}

// Description of the compact plan's pass i (instrumentation): *k, *r = its
// first stage bit and stage count (the low pass last: k = 0, r = w);
// *engine = 32 when the pass runs on the int32 engine (bw_kernels32.cuh), 64
// on the int64 engine's mapped passes; *bytes_per_point = its algorithmic
// bytes (read + write).
int bw_compact_pass_info(int log2n, int pass_index, int* k, int* r, int* engine, int* bytes_per_point) {
    CompactPlan cp;
    if (log2n < 0 || log2n > BW_MAX_LOG2N || !compact_plan(log2n, &cp))
        return fail(BW_BAD_ARGUMENTS, "no compact plan for n = %d", log2n);
    if (pass_index < 0 || pass_index > cp.m) return fail(BW_BAD_ARGUMENTS, "bad compact pass %d", pass_index);
    const Pass& p = cp.pass[pass_index];
    if (k) *k = p.k;
    if (r) *r = p.r;
    if (engine) *engine = cp.v2 && (pass_index > 0 || cp.first32) ? 32 : 64;
    if (bytes_per_point) *bytes_per_point = (pass_index == 0 || pass_index == cp.m) ? 12 : 8;
    return BW_OK;
}

// One pass of the compact plan, asynchronous (benchmark instrumentation):
// checked = 1 runs pass 0 with the input test (then *abort_dev says whether
// it wrote nothing-or-everything; tileflag_dev holds 2^(n-13) words).
int bw_fwht_i64_compact_pass(int64_t* data, int log2n, int pass_index, int checked, uint32_t* tileflag_dev,
                             uint32_t* abort_dev, void* stream) {
    BW_TRY(check_signal(data, log2n));
    CompactPlan cp;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !compact_plan(log2n, &cp))
        return fail(BW_BAD_ARGUMENTS, "no compact plan for this signal (n = %d)", log2n);
    if (pass_index < 0 || pass_index > cp.m) return fail(BW_BAD_ARGUMENTS, "bad compact pass %d", pass_index);
    if (checked && (pass_index != 0 || !tileflag_dev || !abort_dev))
        return fail(BW_BAD_ARGUMENTS, "only pass 0 is checked, with tile flags and an abort word");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    return launch_compact(cp, pass_index, data, checked ? COMPACT_CHECK : COMPACT_PLAIN,
                          reinterpret_cast<unsigned*>(tileflag_dev), reinterpret_cast<unsigned*>(abort_dev),
                          as_stream(stream));
}

// The compact plan's LAST pass (the widening low pass) with the threshold
// extraction fused in, asynchronous (instrumentation; the pass-level form of
// bw_fwht_extract_i64 on small-valued signals).  Needs an int32-engine plan.
int bw_fwht_i64_compact_pass_extract(int64_t* data, int log2n, uint64_t tau, uint64_t base, int64_t* out_idx,
                                     int64_t* out_val, uint64_t cap, uint64_t* count_dev, void* stream) {
    BW_TRY(check_signal(data, log2n));
    if (!count_dev || (cap > 0 && (!out_idx || !out_val))) return fail(BW_BAD_ARGUMENTS, "null extraction output");
    CompactPlan cp;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !compact_plan(log2n, &cp) || !cp.v2)
        return fail(BW_BAD_ARGUMENTS, "no int32-engine compact plan for this signal (n = %d)", log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    bw::ExtractArgs ex = {tau, base, reinterpret_cast<long long*>(out_idx), reinterpret_cast<long long*>(out_val),
                          reinterpret_cast<unsigned long long*>(count_dev), cap};
    return launch_compact(cp, cp.m, data, COMPACT_PLAIN, nullptr, nullptr, as_stream(stream), &ex);
}

// fwht_array with compact in-place intermediates.  max_abs >= 0: the
// caller's bound on |x| (fwht_inplace has just computed it); <= lim(n) runs
// the compact plan unchecked and asynchronously, above it the int64 plan.
// max_abs < 0: unknown -- pass 0 tests every input (synchronises the stream
// once); on a failure the written tiles are restored and the int64 plan runs.
// *used_compact says which plan produced the result (bit-identical anyway).
int bw_fwht_i64_compact(int64_t* data, int log2n, long long max_abs, void* stream, int* used_compact,
                        uint64_t* butterflies) {
    BW_TRY(check_signal(data, log2n));
    if (used_compact) *used_compact = 0;
    if (butterflies) *butterflies = butterfly_count(log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    CompactPlan cp;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !compact_plan(log2n, &cp) || max_abs > cp.lim)
        return fwht_impl(data, log2n, nullptr, false, s);
    if (max_abs >= 0) {
        for (int i = 0; i <= cp.m; ++i) BW_TRY(launch_compact(cp, i, data, COMPACT_PLAIN, nullptr, nullptr, s));
        if (used_compact) *used_compact = 1;
        return BW_OK;
    }
    int used = 0;
    BW_TRY(compact_try(data, log2n, s, &used));
    if (used_compact) *used_compact = used;
    return used ? BW_OK : fwht_impl(data, log2n, nullptr, false, s);
}

// Test hook: restore after a checked pass 0 (the fallback's first step),
// asynchronous.  tileflag_dev / abort_dev as bw_fwht_i64_compact_pass left them.
int bw_fwht_i64_compact_restore(int64_t* data, int log2n, uint32_t* tileflag_dev, void* stream) {
    BW_TRY(check_signal(data, log2n));
    CompactPlan cp;
    if ((reinterpret_cast<uintptr_t>(data) & 15u) || !compact_plan(log2n, &cp) || !tileflag_dev)
        return fail(BW_BAD_ARGUMENTS, "no compact plan for this signal (n = %d) or no tile flags", log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    return launch_compact(cp, 0, data, COMPACT_RESTORE, reinterpret_cast<unsigned*>(tileflag_dev), nullptr,
                          as_stream(stream));
}

}  // extern "C"
namespace {
// ---- the int32 engine (bw_kernels32.cuh): static checks and host emulation
// of its exact tables (TEST HOOKS) -----------------------------------------

// Every round covers the 14 tile bits once (the low pass's sub-rounds: 13
// plus the sub-round bit), stages only register bits, keeps vector accesses
// aligned, and every 4/8/16-byte shared-memory access phase (32 / 16 / 8
// lanes) touches distinct banks.
template <class C, int RD>
bool w32_round_ok(std::string* why) {
    constexpr int NREG = C::nreg(RD);
    uint32_t seen = 0, regs = 0;
    auto add = [&](int b) {
        if (b < 0 || b >= bw::w32::kBits || ((seen >> b) & 1u)) return false;
        seen |= 1u << b;
        return true;
    };
    for (int i = 0; i < NREG; ++i) {
        if (!add(C::reg(RD, i))) { *why = "register bits overlap"; return false; }
        regs |= 1u << C::reg(RD, i);
    }
    for (int i = 0; i < 5; ++i) if (!add(C::lane(RD, i))) { *why = "lane bits overlap"; return false; }
    for (int i = 0; i < 3; ++i) if (!add(C::warp(RD, i))) { *why = "warp bits overlap"; return false; }
    uint32_t sub = 0;
    if constexpr (NREG == 5) {
        sub = 1u << C::SUB;
        if (!add(C::SUB)) { *why = "sub-round bit overlaps"; return false; }
    }
    if (seen != (1u << bw::w32::kBits) - 1u) { *why = "round does not cover the tile"; return false; }
    if (C::stage(RD) & ~regs) { *why = "a staged bit is not a register bit"; return false; }
    constexpr int V = bw::w32::vec<C, RD>();
    constexpr int phase = V == 4 ? 8 : V == 2 ? 16 : 32;
    for (uint32_t s = 0; s < (sub ? 2u : 1u); ++s)
        for (uint32_t warp = 0; warp < 8; ++warp)
            for (int j = 0; j < (1 << NREG); j += V)
                for (uint32_t g0 = 0; g0 < 32; g0 += phase) {
                    uint32_t used = 0;
                    for (uint32_t l = g0; l < g0 + phase; ++l) {
                        const uint32_t e = bw::w32::thread_part<C, RD>(l, warp) | bw::w32::reg_part<C, RD>(j) |
                                           (s ? sub : 0u);
                        const uint32_t slot = C::slot(e);
                        if (slot % V) { *why = "misaligned vector access"; return false; }
                        for (int q = 1; q < V; ++q)
                            if (C::slot(e | bw::w32::reg_part<C, RD>(q)) != slot + q) {
                                *why = "vector elements not consecutive";
                                return false;
                            }
                        for (int q = 0; q < V; ++q) {
                            const uint32_t bank = (slot + q) & 31u;
                            if ((used >> bank) & 1u) { *why = "shared-memory bank conflict"; return false; }
                            used |= 1u << bank;
                        }
                    }
                }
    return true;
}

template <class C, int RD = 0>
bool w32_rounds_ok(std::string* why) {
    if constexpr (RD < C::NR) {
        if (!w32_round_ok<C, RD>(why)) return false;
        return w32_rounds_ok<C, RD + 1>(why);
    }
    return true;
}

// Index of a compact int32 slot (without the half bit).
uint64_t compact_index_of(const Layout& lam, int n, uint64_t slot) {
    uint64_t i = 0;
    for (int b = 0; b < n; ++b)
        if ((slot >> lam.pos[b]) & 1u) i |= 1ull << b;
    return i;
}

// Calls f(phase, tile, e, addr_bytes, width, index) for every element access
// of int32-engine pass q (phase 0: loads in round 0, phase 1: stores in the
// last round) with the kernel's exact address functions.
template <class F>
int w32_visit_pass(const CompactPlan& cp, int q, F&& f) {
    namespace w = bw::w32;
    const Layout lam = compact_layout(cp);
    const int n = cp.n;
    const uint64_t tiles = 1ull << (n - w::kBits);
    const uint64_t so = q > 0 ? (uint64_t)cp.half[q - 1] << cp.w : 0;
    std::string why;
    if (q == cp.m) {
        using C = w::CfgLowW;
        if (!w32_rounds_ok<C>(&why)) return fail(BW_BAD_ARGUMENTS, "int32 low pass layout: %s", why.c_str());
        for (uint64_t b = 0; b < tiles; ++b)
            for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th) {
                const uint32_t lane = th & 31u, warp = th >> 5;
                for (int j = 0; j < w::kE; ++j) {
                    const uint32_t e = w::thread_part<C, 0>(lane, warp) | w::reg_part<C, 0>(j);
                    // the kernel treats tile element e as index (b << 14) + e
                    const uint64_t slot = (b << (w::kBits + 1)) + C::src_off(e);
                    f(0, b, e, (so + slot) * 4, 4, (b << w::kBits) + e);
                }
                for (uint32_t s = 0; s < 2; ++s)
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t e = w::thread_part<C, 2>(lane, warp) | (s << C::SUB) | w::reg_part<C, 2>(j);
                        const uint64_t gi = (b << w::kBits) + e;
                        f(1, b, e, gi * 8, 8, gi);
                    }
            }
        return BW_OK;
    }
    const Pass& p = cp.pass[q];
    const uint64_t dof = (uint64_t)cp.half[q] << cp.w;
    if (q > 0 && p.r >= 1 && p.r <= 4) {  // k32_reg: every thread's 4 slots of every row, read half -> write half
        const int kk = p.k + 1, R = p.r;
        const uint64_t threads = 1ull << (n - R - 2);
        for (uint64_t th = 0; th < threads; ++th) {
            const uint64_t base = R == 1 ? w::reg_slot_base<1>(th * 4, kk) : R == 2 ? w::reg_slot_base<2>(th * 4, kk)
                                  : R == 3 ? w::reg_slot_base<3>(th * 4, kk) : w::reg_slot_base<4>(th * 4, kk);
            for (uint64_t r = 0; r < (1ull << R); ++r)
                for (uint64_t c = 0; c < 4; ++c) {
                    const uint64_t sl = base + (r << kk) + c;
                    const uint64_t gi = compact_index_of(lam, n, sl);
                    if (c == 0 && (compact_index_of(lam, n, base + (r << kk)) ^ compact_index_of(lam, n, base)) != (r << p.k))
                        return fail(BW_BAD_ARGUMENTS, "int32 register pass: row %llu is not at index bit %d", (unsigned long long)r, p.k);
                    f(0, th / w::kNT, (uint32_t)(r * 4 + c), (so + sl) * 4, 4, gi);
                    f(1, th / w::kNT, (uint32_t)(r * 4 + c), (dof + sl) * 4, 4, gi);
                }
        }
        return BW_OK;
    }
    auto run = [&](auto cfg, auto lc) -> int {
        using C = typename decltype(cfg)::type;
        constexpr int L = decltype(lc)::value;
        if (!w32_rounds_ok<C>(&why)) return fail(BW_BAD_ARGUMENTS, "int32 high pass layout: %s", why.c_str());
        const int kk = p.k + 1;
        for (int i = 0; i < p.r; ++i)  // tile row i is index bit k + i (the stage the kernel applies)
            if (compact_index_of(lam, n, w::high_off<L>(1u << (L + i), kk)) != 1ull << (p.k + i))
                return fail(BW_BAD_ARGUMENTS, "int32 high pass row %d is not index bit %d", i, p.k + i);
        for (uint64_t t = 0; t < tiles; ++t) {
            const uint64_t base = w::high_tile_base<L>(t, kk);
            for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th) {
                const uint32_t lane = th & 31u, warp = th >> 5;
                for (int j = 0; j < w::kE; ++j) {
                    const uint32_t ei = w::thread_part<C, 0>(lane, warp) | w::reg_part<C, 0>(j);
                    const uint64_t si = base + w::high_off<L>(ei, kk);
                    if (q == 0) {  // k32_first: the natural int64 element (k32_restore stores the same addresses)
                        const uint64_t gi = w::first_base(base) + w::first_off<L>(ei, p.k);
                        if (gi != compact_index_of(lam, n, si)) return fail(BW_BAD_ARGUMENTS, "first pass: natural / compact tile maps differ");
                        f(0, t, ei, gi * 8, 8, gi);
                    } else
                        f(0, t, ei, (so + si) * 4, 4, compact_index_of(lam, n, si));
                    const uint32_t eo = w::thread_part<C, 1>(lane, warp) | w::reg_part<C, 1>(j);
                    const uint64_t sd = base + w::high_off<L>(eo, kk);
                    f(1, t, eo, (dof + sd) * 4, 4, compact_index_of(lam, n, sd));
                }
            }
        }
        return BW_OK;
    };
    if (p.r == 9) return run(tag<w::CfgHighW<5>>{}, ic<5>{});
    if (p.r == 8) return run(tag<w::CfgHighW<6>>{}, ic<6>{});
    if (p.r == 7 && q > 0) return run(tag<w::CfgHighW<7>>{}, ic<7>{});
    if (p.r == 6 && q > 0) return run(tag<w::CfgHighW<8>>{}, ic<8>{});
    return fail(BW_BAD_ARGUMENTS, "no int32-engine pass of %d rows", p.r);
}

// Host emulation of the compact plan with its int32-engine passes (TEST
// HOOK): pass 0 by its definition (its rows' stages, then the int32 store
// into the compact layout), every later pass thread by thread with the
// kernels' own tables, rounds, swizzled shared-memory slots and int32 /
// int64 arithmetic.
int w32_emulate(int64_t* host, const CompactPlan& cp) {
    namespace w = bw::w32;
    const int n = cp.n;
    const uint64_t N = 1ull << n;
    const Layout lam = compact_layout(cp);
    std::vector<uint32_t> buf(2 * N);
    memcpy(buf.data(), host, 8 * N);
    if (!cp.first32) {  // pass 0: rows [w, w + r) staged on the int64 values, stored as int32
        std::vector<u64> x(N);
        memcpy(x.data(), host, 8 * N);
        const Pass& p = cp.pass[0];
        for (int k = p.k; k < p.k + p.r; ++k)
            for (uint64_t i = 0; i < N; ++i)
                if (!((i >> k) & 1)) {
                    const u64 a = x[i], b = x[i | (1ull << k)];
                    x[i] = a + b;
                    x[i | (1ull << k)] = a - b;
                }
        const uint64_t dof = (uint64_t)cp.half[0] << cp.w;
        for (uint64_t i = 0; i < N; ++i) {
            uint64_t slot = 0;
            for (int b = 0; b < n; ++b)
                if ((i >> b) & 1) slot |= 1ull << lam.pos[b];
            buf[dof + slot] = (uint32_t)x[i];
        }
    }
    std::vector<uint32_t> v((size_t)w::kNT * w::kE), sm(1u << w::kBits);
    auto stages32 = [&](auto cfg, auto rdc) {
        using C = typename decltype(cfg)::type;
        constexpr int RD = decltype(rdc)::value;
        for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
            for (int i = 0; i < C::nreg(RD); ++i)
                if ((C::stage(RD) >> C::reg(RD, i)) & 1u)
                    for (int j = 0; j < w::kE; ++j)
                        if (!((j >> i) & 1)) {
                            uint32_t& a = v[th * w::kE + j];
                            uint32_t& b = v[th * w::kE + (j | (1 << i))];
                            const uint32_t x = a, y = b;
                            a = x + y;
                            b = x - y;
                        }
    };
    auto to_smem = [&](auto cfg, auto rdc) {
        using C = typename decltype(cfg)::type;
        constexpr int RD = decltype(rdc)::value;
        for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
            for (int j = 0; j < w::kE; ++j)
                sm[C::slot(w::thread_part<C, RD>(th & 31u, th >> 5) | w::reg_part<C, RD>(j))] = v[th * w::kE + j];
    };
    auto from_smem = [&](auto cfg, auto rdc) {
        using C = typename decltype(cfg)::type;
        constexpr int RD = decltype(rdc)::value;
        for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
            for (int j = 0; j < w::kE; ++j)
                v[th * w::kE + j] = sm[C::slot(w::thread_part<C, RD>(th & 31u, th >> 5) | w::reg_part<C, RD>(j))];
    };
    const uint64_t tiles = 1ull << (n - w::kBits);
    for (int q = cp.first32 ? 0 : 1; q <= cp.m; ++q) {
        const uint64_t so = q > 0 ? (uint64_t)cp.half[q - 1] << cp.w : 0;
        if (q == cp.m) {
            using C = w::CfgLowW;
            for (uint64_t b = 0; b < tiles; ++b) {
                for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
                    for (int j = 0; j < w::kE; ++j)
                        v[th * w::kE + j] = buf[so + (b << (w::kBits + 1)) +
                                                C::src_off(w::thread_part<C, 0>(th & 31u, th >> 5) | w::reg_part<C, 0>(j))];
                stages32(tag<C>{}, ic<0>{});
                to_smem(tag<C>{}, ic<0>{});
                from_smem(tag<C>{}, ic<1>{});
                stages32(tag<C>{}, ic<1>{});
                to_smem(tag<C>{}, ic<1>{});
                for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
                    for (uint32_t s = 0; s < 2; ++s) {
                        const uint32_t tp = w::thread_part<C, 2>(th & 31u, th >> 5) | (s << C::SUB);
                        u64 x[32];
                        for (int j = 0; j < 32; ++j) x[j] = (u64)(int64_t)(int32_t)sm[C::slot(tp | w::reg_part<C, 2>(j))];
                        for (int i = 0; i < 5; ++i)
                            if ((C::stage(2) >> C::reg(2, i)) & 1u)
                                for (int j = 0; j < 32; ++j)
                                    if (!((j >> i) & 1)) {
                                        const u64 a = x[j], c = x[j | (1 << i)];
                                        x[j] = a + c;
                                        x[j | (1 << i)] = a - c;
                                    }
                        for (int j = 0; j < 32; ++j) {
                            const uint64_t gi = (b << w::kBits) + (tp | w::reg_part<C, 2>(j));
                            buf[2 * gi] = (uint32_t)x[j];
                            buf[2 * gi + 1] = (uint32_t)(x[j] >> 32);
                        }
                    }
            }
            continue;
        }
        const Pass& p = cp.pass[q];
        const uint64_t dof = (uint64_t)cp.half[q] << cp.w;
        if (q > 0 && p.r >= 1 && p.r <= 4) {  // k32_reg, thread by thread
            const int kk = p.k + 1, R = p.r;
            for (uint64_t th = 0; th < (1ull << (n - R - 2)); ++th) {
                const uint64_t base = R == 1 ? w::reg_slot_base<1>(th * 4, kk) : R == 2 ? w::reg_slot_base<2>(th * 4, kk)
                                      : R == 3 ? w::reg_slot_base<3>(th * 4, kk) : w::reg_slot_base<4>(th * 4, kk);
                for (uint64_t c = 0; c < 4; ++c) {
                    uint32_t x[16];
                    for (uint64_t r = 0; r < (1ull << R); ++r) x[r] = buf[so + base + (r << kk) + c];
                    for (int i = 0; i < R; ++i)
                        for (uint64_t r = 0; r < (1ull << R); ++r)
                            if (!((r >> i) & 1)) {
                                const uint32_t a = x[r], b = x[r | (1ull << i)];
                                x[r] = a + b;
                                x[r | (1ull << i)] = a - b;
                            }
                    for (uint64_t r = 0; r < (1ull << R); ++r) buf[dof + base + (r << kk) + c] = x[r];
                }
            }
            continue;
        }
        auto run = [&](auto cfg, auto lc) {
            using C = typename decltype(cfg)::type;
            constexpr int L = decltype(lc)::value;
            const int kk = p.k + 1;
            for (uint64_t t = 0; t < tiles; ++t) {
                const uint64_t base = w::high_tile_base<L>(t, kk);
                for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
                    for (int j = 0; j < w::kE; ++j) {
                        const uint32_t e = w::thread_part<C, 0>(th & 31u, th >> 5) | w::reg_part<C, 0>(j);
                        // k32_first keeps the low word of the natural int64 element (little endian)
                        v[th * w::kE + j] = q == 0 ? buf[2 * (w::first_base(base) + w::first_off<L>(e, p.k))]
                                                   : buf[so + base + w::high_off<L>(e, kk)];
                    }
                stages32(tag<C>{}, ic<0>{});
                to_smem(tag<C>{}, ic<0>{});
                from_smem(tag<C>{}, ic<1>{});
                stages32(tag<C>{}, ic<1>{});
                for (uint32_t th = 0; th < (uint32_t)w::kNT; ++th)
                    for (int j = 0; j < w::kE; ++j)
                        buf[dof + base + w::high_off<L>(w::thread_part<C, 1>(th & 31u, th >> 5) | w::reg_part<C, 1>(j), kk)] =
                            v[th * w::kE + j];
            }
        };
        if (p.r == 9) run(tag<w::CfgHighW<5>>{}, ic<5>{});
        else if (p.r == 8) run(tag<w::CfgHighW<6>>{}, ic<6>{});
        else if (p.r == 7 && q > 0) run(tag<w::CfgHighW<7>>{}, ic<7>{});
        else if (p.r == 6 && q > 0) run(tag<w::CfgHighW<8>>{}, ic<8>{});
        else return fail(BW_BAD_ARGUMENTS, "no int32-engine pass of %d rows", p.r);
    }
    memcpy(host, buf.data(), 8 * N);
    return BW_OK;
}
}  // namespace
extern "C" {

// TEST HOOK ONLY: host emulation of the compact plan (v2: its int32-engine
// passes run thread by thread from the kernels' tables), 16 <= n <= 24.
int bw_debug_emulate_compact(int64_t* host, int log2n) {
    if (!host || log2n < 16 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "compact emulation supports 16 <= n <= 24");
    CompactPlan cp;
    if (!compact_plan(log2n, &cp) || !cp.v2) return fail(BW_BAD_ARGUMENTS, "no int32-engine compact plan for n = %d", log2n);
    return w32_emulate(host, cp);
}

// Static checker of the compact plan (TEST HOOK, 16 <= n <= 24): runs the
// kernels' exact address tables for every element of every pass and checks
//   - pass 0 loads natural int64, the last pass stores natural int64;
//   - pass i+1 loads every element at the bytes (and width) pass i stored it;
//   - no two stores of a pass overlap, every access stays in the buffer;
//   - IN PLACE: no tile stores into bytes another tile of the same pass
//     loads (4-byte granules; cluster tiles count as one tile);
//   - every index bit is staged by exactly one pass.
int bw_plan_check_compact(int log2n) {
    if (log2n < 16 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "compact plan check supports 16 <= n <= 24");
    CompactPlan cp;
    if (!compact_plan(log2n, &cp)) return fail(BW_BAD_ARGUMENTS, "no compact plan for n = %d", log2n);
    const uint64_t N = 1ull << log2n, G = 2 * N;  // 4-byte granules of the buffer
    const Layout nat = natural_layout(log2n), lam = compact_layout(cp);
    std::vector<uint64_t> ld(N), st(N), prev(N);
    std::vector<uint8_t> ldw(N), stw(N), prevw(N);
    std::vector<int32_t> reader(G), writer(G);
    uint64_t staged = 0;
    auto base_of = [](const bw::LayoutTab& t, uint64_t tile, uint32_t vt) {
        unsigned long long off = 0;
        for (int r = 0; r < t.nruns; ++r) off += ((tile >> t.rsrc[r]) & ((1ull << t.rlen[r]) - 1ull)) << t.rdst[r];
        for (int b = 0; b < 16; ++b)
            if ((vt >> b) & 1u) off += t.bit[b];
        return off;
    };
    for (int q = 0; q <= cp.m; ++q) {
        int ok;
        if (cp.v2 && (q > 0 || cp.first32)) {  // the int32 engine's exact address functions
            std::fill(reader.begin(), reader.end(), -1);
            std::fill(writer.begin(), writer.end(), -1);
            const Pass& p = cp.pass[q];
            const uint64_t bits = q == cp.m ? (1ull << cp.w) - 1ull : ((1ull << p.r) - 1ull) << p.k;
            if (staged & bits) return fail(BW_BAD_ARGUMENTS, "pass %d stages a bit twice", q);
            staged |= bits;
            const char* err = nullptr;
            ok = w32_visit_pass(cp, q, [&](int phase, uint64_t tile, uint32_t, uint64_t a, int width, uint64_t gi) {
                if (gi >= N || a + width > 8 * N) { err = "an access leaves the buffer"; return; }
                if (phase == 0) {
                    ld[gi] = a;
                    ldw[gi] = (uint8_t)width;
                    for (uint64_t gr = a / 4; gr < (a + width) / 4; ++gr) reader[gr] = (int32_t)tile;
                } else {
                    st[gi] = a;
                    stw[gi] = (uint8_t)width;
                }
            });
            if (ok == BW_OK) {  // stores checked after every load of the pass is known
                ok = w32_visit_pass(cp, q, [&](int phase, uint64_t tile, uint32_t, uint64_t a, int width, uint64_t) {
                    if (phase != 1) return;
                    for (uint64_t gr = a / 4; gr < (a + width) / 4; ++gr) {
                        if (writer[gr] != -1) { err = "two stores to one granule"; return; }
                        writer[gr] = (int32_t)tile;
                        if (reader[gr] != -1 && reader[gr] != (int32_t)tile) { err = "a tile stores over bytes another tile loads (not in place)"; return; }
                    }
                });
            }
            if (ok == BW_OK && err) return fail(BW_BAD_ARGUMENTS, "pass %d: %s", q, err);
        } else ok = visit_compact(cp.pass[q], [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            constexpr int NQ = 1 << C::Q, LAST = C::NR - 1;
            const PassGeom& g = cp.geom[q];
            const bool low = q == cp.m;
            // source / destination: layout, element bytes, element offset of the pointer
            const Layout& sl = q == 0 ? nat : lam;
            const Layout& dl = low ? nat : lam;
            const int sb = q == 0 ? 8 : 4, db = low ? 8 : 4;
            const uint64_t so = q == 0 ? 0 : (uint64_t)cp.half[q - 1] << cp.w;
            const uint64_t dof = low ? 0 : (uint64_t)cp.half[q] << cp.w;
            bw::LayoutTab tl, ts, tgi, tgo;
            fill_layout_tab<C, 0>(g, log2n, sl, &tl);
            fill_layout_tab<C, LAST>(g, log2n, dl, &ts);
            fill_layout_tab<C, 0>(g, log2n, nat, &tgi);  // global index of the loaded element
            fill_layout_tab<C, LAST>(g, log2n, nat, &tgo);
            for (int vb = L >= C::T ? 0 : L; vb < C::T; ++vb) {  // a low pass stages its whole tile
                if ((staged >> g.gb[vb]) & 1) return fail(BW_BAD_ARGUMENTS, "bit %d staged twice", g.gb[vb]);
                staged |= 1ull << g.gb[vb];
            }
            std::fill(reader.begin(), reader.end(), -1);
            std::fill(writer.begin(), writer.end(), -1);
            const uint64_t ctas = 1ull << (log2n - bw::kCtaBits);
            for (int phase = 0; phase < 2; ++phase) {  // loads first (owners), then stores
                for (uint64_t cta = 0; cta < ctas; ++cta) {
                    const uint32_t rank = (uint32_t)(cta & (NQ - 1));
                    const int32_t tile = (int32_t)(cta >> C::Q);
                    for (uint32_t th = 0; th < (uint32_t)bw::Dims<C>::NT; ++th) {
                        const uint32_t lane = th & 31u, warp = th >> 5;
                        const uint32_t v0 = bw::thread_part<C, 0>(lane, warp) | bw::rank_bits<C, 0>(rank);
                        const uint32_t v1 = bw::thread_part<C, LAST>(lane, warp) | bw::rank_bits<C, LAST>(rank);
                        for (int j = 0; j < bw::Dims<C>::E; ++j) {
                            if (phase == 0) {
                                const uint64_t gi = base_of(tgi, tile, v0) + tgi.reg[j];
                                const uint64_t a = (so + base_of(tl, tile, v0) + tl.reg[j]) * sb;
                                if (gi >= N || a + sb > 8 * N) return fail(BW_BAD_ARGUMENTS, "pass %d loads outside", q);
                                ld[gi] = a;
                                ldw[gi] = (uint8_t)sb;
                                for (uint64_t gr = a / 4; gr < (a + sb) / 4; ++gr) reader[gr] = tile;
                            } else {
                                const uint64_t go = base_of(tgo, tile, v1) + tgo.reg[j];
                                const uint64_t a = (dof + base_of(ts, tile, v1) + ts.reg[j]) * db;
                                if (go >= N || a + db > 8 * N) return fail(BW_BAD_ARGUMENTS, "pass %d stores outside", q);
                                st[go] = a;
                                stw[go] = (uint8_t)db;
                                for (uint64_t gr = a / 4; gr < (a + db) / 4; ++gr) {
                                    if (writer[gr] != -1) return fail(BW_BAD_ARGUMENTS, "pass %d stores twice", q);
                                    writer[gr] = tile;
                                    if (reader[gr] != -1 && reader[gr] != tile)
                                        return fail(BW_BAD_ARGUMENTS,
                                                    "pass %d: tile %lld stores over bytes tile %lld loads (not in place)",
                                                    q, (long long)tile, (long long)reader[gr]);
                                }
                            }
                        }
                    }
                }
            }
            return BW_OK;
        });
        if (ok != BW_OK) return ok;
        for (uint64_t i = 0; i < N; ++i) {
            if (q == 0 && (ld[i] != 8 * i || ldw[i] != 8)) return fail(BW_BAD_ARGUMENTS, "pass 0 does not load natural int64");
            if (q > 0 && (ld[i] != prev[i] || ldw[i] != prevw[i]))
                return fail(BW_BAD_ARGUMENTS, "pass %d loads index %llu elsewhere", q, (unsigned long long)i);
            if (q == cp.m && (st[i] != 8 * i || stw[i] != 8))
                return fail(BW_BAD_ARGUMENTS, "last pass does not store natural int64");
        }
        prev.swap(st);
        prevw.swap(stw);
    }
    if (staged != N - 1) return fail(BW_BAD_ARGUMENTS, "stages cover 0x%llx, not every bit", (unsigned long long)staged);
    return BW_OK;
}

}  // extern "C"
namespace {
// Host buffer -> device -> host with the copies overlapping the passes:
// the H2D of each chunk is followed at once by the passes that stay inside
// a chunk (every pass but the last), and the last pass runs in column
// slices, each slice's rows going back with a 2-D D2H copy while the next
// slice computes.  Copies run on a per-device copy stream, ordered against
// the caller's stream with events.  *done = false when the plan does not
// have that shape (the caller then runs the plain sequence).
cudaStream_t g_copy_stream[kMaxDevices];
cudaStream_t g_d2h_stream[kMaxDevices];

// Geometry of a copy-overlapped host transform: one-run passes, the H2D in
// <= 128 chunks of 2^cb points each followed by the passes that stay inside
// a chunk (every pass but the last), the last pass in 16 column slices of
// 2^wb columns, each sliced out with a 2-D D2H.  ok = false: no such shape.
struct HostPipe {
    bool ok = false;
    std::vector<Pass> passes;
    int B = 0, cb = 0, wb = 0, nchunks = 0, nslices = 0;
};

int host_pipe_plan(int log2n, HostPipe* hp) {
    hp->ok = false;
    if (log2n < 24) return BW_OK;
    std::vector<int> w;
    // one-run passes: every pass but the last stays inside a chunk (a split
    // pass would reach the top bits; the overlap saves far more, ~65 ms at
    // n = 32, than the split plan's 0.8 ms)
    BW_TRY(default_plan(log2n, &w, true));
    BW_TRY(build_passes(log2n, w, &hp->passes));
    const std::vector<Pass>& passes = hp->passes;
    if (passes.size() < 2) return BW_OK;
    const Pass last = passes.back();
    if ((last.kind != HIGH && last.kind != REG) || last.a || last.k + last.r != log2n) return BW_OK;
    for (const Pass& p : passes)
        if (p.a) return BW_OK;  // split rows leave a chunk
    const int B = last.k;                                  // the other passes cover stages [0, B)
    const int cb = B > log2n - 7 ? B : log2n - 7;          // H2D chunks of 2^cb points (<= 128 chunks)
    const int wb = B - 4;                                  // last pass in 16 column slices of 2^wb columns
    int colbits = 0;
    BW_TRY(visit_pass(last, [&](auto t, auto l) -> int {
        colbits = decltype(l)::value;
        return BW_OK;
    }));
    if (wb < colbits || wb + last.r < bw::kCtaBits + last.q) return BW_OK;
    hp->B = B;
    hp->cb = cb;
    hp->wb = wb;
    hp->nchunks = 1 << (log2n - cb);
    hp->nslices = 1 << (B - wb);
    hp->ok = true;
    return BW_OK;
}

int host_pipelined(int64_t* host, int log2n, u64* d, int dev, cudaStream_t s, bool* done) {
    *done = false;
    HostPipe hp;
    BW_TRY(host_pipe_plan(log2n, &hp));
    if (!hp.ok) return BW_OK;
    const std::vector<Pass>& passes = hp.passes;
    const Pass last = passes.back();
    const int B = hp.B, cb = hp.cb, wb = hp.wb, nchunks = hp.nchunks, nslices = hp.nslices;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_copy_stream[dev]) BW_CUDA(cudaStreamCreateWithFlags(&g_copy_stream[dev], cudaStreamNonBlocking));
    }
    cudaStream_t cs = g_copy_stream[dev];
    std::vector<cudaEvent_t> ev(nchunks + nslices + 2);
    for (auto& e : ev) BW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const int st = [&]() -> int {
        BW_CUDA(cudaEventRecord(ev[0], s));  // the copy stream follows earlier work on the caller's stream
        BW_CUDA(cudaStreamWaitEvent(cs, ev[0], 0));
        for (int c = 0; c < nchunks; ++c) {
            const size_t off = (size_t)c << cb;
            BW_CUDA(cudaMemcpyAsync(d + off, host + off, (size_t)8 << cb, cudaMemcpyHostToDevice, cs));
            BW_CUDA(cudaEventRecord(ev[1 + c], cs));
            BW_CUDA(cudaStreamWaitEvent(s, ev[1 + c], 0));
            for (size_t i = 0; i + 1 < passes.size(); ++i) BW_TRY(launch_pass(passes[i], d + off, cb, s));
        }
        for (int j = 0; j < nslices; ++j) {
            const size_t off = (size_t)j << wb;
            BW_TRY(launch_pass(last, d + off, wb + last.r, s));
            BW_CUDA(cudaEventRecord(ev[1 + nchunks + j], s));
            BW_CUDA(cudaStreamWaitEvent(cs, ev[1 + nchunks + j], 0));
            BW_CUDA(cudaMemcpy2DAsync(host + off, (size_t)8 << B, d + off, (size_t)8 << B, (size_t)8 << wb,
                                      (size_t)1 << last.r, cudaMemcpyDeviceToHost, cs));
        }
        BW_CUDA(cudaEventRecord(ev.back(), cs));
        BW_CUDA(cudaStreamWaitEvent(s, ev.back(), 0));
        return BW_OK;
    }();
    BW_CUDA(cudaStreamSynchronize(s));
    for (auto& e : ev) cudaEventDestroy(e);
    if (st != BW_OK) return st;
    *done = true;
    return BW_OK;
}
}  // namespace
extern "C" {

int bw_fwht_host_i64(int64_t* host, int log2n, int64_t* work_dev, int check_bound, void* stream,
                     uint64_t* butterflies) {
    if (!host) return fail(BW_BAD_ARGUMENTS, "null host pointer");
    BW_TRY(check_signal(work_dev, log2n));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    if (!check_bound && !(reinterpret_cast<uintptr_t>(work_dev) & 15u) && g_host_pipeline) {
        bool done = false;
        BW_TRY(host_pipelined(host, log2n, reinterpret_cast<u64*>(work_dev), dev, s, &done));
        if (done) {
            if (butterflies) *butterflies = butterfly_count(log2n);
            return BW_OK;
        }
    }
    const size_t bytes = (size_t)8 << log2n;
    BW_CUDA(cudaMemcpyAsync(work_dev, host, bytes, cudaMemcpyHostToDevice, s));
    int64_t* sc = nullptr;
    if (check_bound) {
        void* p = nullptr;
        BW_TRY(scratch(dev, 64, &p));
        sc = reinterpret_cast<int64_t*>(p);
        BW_TRY(minmax_impl(work_dev, 1ull << log2n, sc, dev, s));
    }
    BW_TRY(fwht_impl(work_dev, log2n, nullptr, false, s));
    if (check_bound) {
        int64_t mm[2];
        BW_CUDA(cudaMemcpyAsync(mm, sc, sizeof mm, cudaMemcpyDeviceToHost, s));
        BW_CUDA(cudaStreamSynchronize(s));
        const uint64_t M = magnitude(mm[0], mm[1]);
        if (!bound_ok(M, log2n))
            return fail(BW_OVERFLOW_BOUND,
                        "max |x| = %llu with n = %d can overflow int64; need |x| * 2**n < 2**63",
                        (unsigned long long)M, log2n);
    }
    BW_CUDA(cudaMemcpyAsync(host, work_dev, bytes, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (butterflies) *butterflies = butterfly_count(log2n);
    return BW_OK;
}

// A batch of host signals, each transformed like bw_fwht_host_i64: the
// signals rotate over nwork device buffers, so signal i+1's H2D runs
// while signal i's D2H runs (PCIe is full duplex; one signal alone cannot
// overlap them, since no output is final before every input has arrived).
// H2D, transforms and D2H run on three streams ordered by events.  A host
// buffer listed twice in a row is processed in order (its second H2D waits
// for the first D2H), so the list behaves like fwht_array on each entry.
int bw_fwht_host_batch_i64(int64_t* const* host, int count, int log2n, int64_t* const* work, int nwork,
                           void* stream, uint64_t* butterflies) {
    if (!host || count < 0) return fail(BW_BAD_ARGUMENTS, "bad host signal list");
    for (int i = 0; i < count; ++i)
        if (!host[i]) return fail(BW_BAD_ARGUMENTS, "null host signal %d", i);
    if (!work || nwork < 1 || nwork > 4) return fail(BW_BAD_ARGUMENTS, "1 to 4 device work buffers");
    for (int b = 0; b < nwork; ++b) {
        BW_TRY(check_signal(work[b], log2n));
        for (int c = 0; c < b; ++c)
            if (work[c] == work[b]) return fail(BW_BAD_ARGUMENTS, "the device work buffers must differ");
    }
    if (butterflies) *butterflies = butterfly_count(log2n);
    if (count == 0) return BW_OK;
    if (count == 1 || nwork == 1) {
        for (int i = 0; i < count; ++i) BW_TRY(bw_fwht_host_i64(host[i], log2n, work[0], 0, stream, nullptr));
        return BW_OK;
    }
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_copy_stream[dev]) BW_CUDA(cudaStreamCreateWithFlags(&g_copy_stream[dev], cudaStreamNonBlocking));
        if (!g_d2h_stream[dev]) BW_CUDA(cudaStreamCreateWithFlags(&g_d2h_stream[dev], cudaStreamNonBlocking));
    }
    cudaStream_t up = g_copy_stream[dev], down = g_d2h_stream[dev];
    const size_t bytes = (size_t)8 << log2n;
    const int nb = nwork;
    cudaEvent_t start, loaded[4], done[4], freed[4];
    // BW_BATCH_PIPELINE=0: whole-signal copies around each transform (A/B knob)
    HostPipe hp;
    BW_TRY(host_pipe_plan(log2n, &hp));
    const bool pipe = hp.ok && g_host_pipeline && !(getenv("BW_BATCH_PIPELINE") && getenv("BW_BATCH_PIPELINE")[0] == '0') &&
                      !(reinterpret_cast<uintptr_t>(work[0]) & 15u) && !(reinterpret_cast<uintptr_t>(work[nwork - 1]) & 15u);
    std::vector<cudaEvent_t> chunk_ev(pipe ? hp.nchunks : 0), slice_ev(pipe ? hp.nslices : 0);
    for (auto& e : chunk_ev) BW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : slice_ev) BW_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    BW_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    for (int b = 0; b < nb; ++b) {
        BW_CUDA(cudaEventCreateWithFlags(&loaded[b], cudaEventDisableTiming));
        BW_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
        BW_CUDA(cudaEventCreateWithFlags(&freed[b], cudaEventDisableTiming));
    }
    const int st = [&]() -> int {
        BW_CUDA(cudaEventRecord(start, s));  // the copies follow earlier work on the caller's stream
        BW_CUDA(cudaStreamWaitEvent(up, start, 0));
        for (int i = 0; i < count; ++i) {
            const int b = i % nb;
            if (i >= nb) BW_CUDA(cudaStreamWaitEvent(up, freed[b], 0));  // signal i-nb's D2H left this buffer
            // Host memory read here and written back by a signal whose D2H
            // may still be in flight (i-nb+1 .. i-1; i-nb and earlier are
            // ordered by freed[b] above, the D2H stream being in order):
            // wait for the latest such D2H, which implies the earlier ones.
            const char* hi = reinterpret_cast<const char*>(host[i]);
            for (int j = i - 1; j > i - nb && j >= 0; --j) {
                const char* hj = reinterpret_cast<const char*>(host[j]);
                if (hi < hj + bytes && hj < hi + bytes) {
                    BW_CUDA(cudaStreamWaitEvent(up, freed[j % nb], 0));
                    break;
                }
            }
            if (pipe) {
                // chunked H2D, each chunk's inner passes as soon as it lands;
                // the last pass in column slices, each slice's D2H right after
                // it: the transform hides under the copies of its neighbours
                u64* d = reinterpret_cast<u64*>(work[b]);
                for (int c = 0; c < hp.nchunks; ++c) {
                    const size_t off = (size_t)c << hp.cb;
                    BW_CUDA(cudaMemcpyAsync(d + off, host[i] + off, (size_t)8 << hp.cb, cudaMemcpyHostToDevice, up));
                    BW_CUDA(cudaEventRecord(chunk_ev[c], up));
                    BW_CUDA(cudaStreamWaitEvent(s, chunk_ev[c], 0));
                    for (size_t q = 0; q + 1 < hp.passes.size(); ++q) BW_TRY(launch_pass(hp.passes[q], d + off, hp.cb, s));
                }
                const Pass& last = hp.passes.back();
                for (int j = 0; j < hp.nslices; ++j) {
                    const size_t off = (size_t)j << hp.wb;
                    BW_TRY(launch_pass(last, d + off, hp.wb + last.r, s));
                    BW_CUDA(cudaEventRecord(slice_ev[j], s));
                    BW_CUDA(cudaStreamWaitEvent(down, slice_ev[j], 0));
                    BW_CUDA(cudaMemcpy2DAsync(host[i] + off, (size_t)8 << hp.B, d + off, (size_t)8 << hp.B,
                                              (size_t)8 << hp.wb, (size_t)1 << last.r, cudaMemcpyDeviceToHost, down));
                }
                BW_CUDA(cudaEventRecord(freed[b], down));
                continue;
            }
            BW_CUDA(cudaMemcpyAsync(work[b], host[i], bytes, cudaMemcpyHostToDevice, up));
            BW_CUDA(cudaEventRecord(loaded[b], up));
            BW_CUDA(cudaStreamWaitEvent(s, loaded[b], 0));
            BW_TRY(fwht_impl(work[b], log2n, nullptr, false, s));
            BW_CUDA(cudaEventRecord(done[b], s));
            BW_CUDA(cudaStreamWaitEvent(down, done[b], 0));
            BW_CUDA(cudaMemcpyAsync(host[i], work[b], bytes, cudaMemcpyDeviceToHost, down));
            BW_CUDA(cudaEventRecord(freed[b], down));
        }
        for (int b = 0; b < nb && b < count; ++b) BW_CUDA(cudaStreamWaitEvent(s, freed[b], 0));
        return BW_OK;
    }();
    BW_CUDA(cudaStreamSynchronize(s));
    cudaEventDestroy(start);
    for (int b = 0; b < nb; ++b) {
        cudaEventDestroy(loaded[b]);
        cudaEventDestroy(done[b]);
        cudaEventDestroy(freed[b]);
    }
    for (auto& e : chunk_ev) cudaEventDestroy(e);
    for (auto& e : slice_ev) cudaEventDestroy(e);
    return st;
}

// ---- out-of-core transform of a host array (external.py:65-283) ----------
//
// The paper's blocked external algorithm with the GPU as the in-memory
// engine and host memory as the "disk": pass 0 transforms contiguous chunks
// of 2^cb elements (_initial_pass, external.py:238-254, with 2^B = chunk);
// each following pass takes g <= cb - 13 consecutive high bits [k, k+g) and
// moves 2^g rows x 64 KiB columns per chunk with 2-D copies (the paper's
// _blocked_stage_pass, external.py:272-283, but g stages per pass instead of
// one).  Two streams alternate over the two halves of the workspace, so one
// chunk's H2D overlaps the other's transform and D2H.
namespace {
cudaStream_t g_ooc_streams[kMaxDevices][2];
int ooc_streams(int dev, cudaStream_t* out) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (int i = 0; i < 2; ++i) {
        if (!g_ooc_streams[dev][i]) {
            cudaError_t e = cudaStreamCreateWithFlags(&g_ooc_streams[dev][i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
        out[i] = g_ooc_streams[dev][i];
    }
    return BW_OK;
}
}  // namespace

int bw_fwht_host_ooc_i64(int64_t* host, int log2n, int64_t* work_dev, int log2_work, void* stream,
                         int* host_passes) {
    if (!host) return fail(BW_BAD_ARGUMENTS, "null host pointer");
    BW_TRY(check_signal(work_dev, log2_work));
    if (reinterpret_cast<uintptr_t>(work_dev) & 15u) return fail(BW_BAD_ARGUMENTS, "workspace must be 16-byte aligned");
    if (log2n < 0 || log2n > 40) return fail(BW_BAD_ARGUMENTS, "log2n = %d outside 0..40", log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t caller = as_stream(stream);
    const int cb = log2_work - 1;  // two half-workspaces of 2^cb elements
    if (log2n <= log2_work) {  // fits: one in-memory transform
        const size_t bytes = (size_t)8 << log2n;
        BW_CUDA(cudaMemcpyAsync(work_dev, host, bytes, cudaMemcpyHostToDevice, caller));
        BW_TRY(fwht_impl(work_dev, log2n, nullptr, false, caller));
        BW_CUDA(cudaMemcpyAsync(host, work_dev, bytes, cudaMemcpyDeviceToHost, caller));
        BW_CUDA(cudaStreamSynchronize(caller));
        if (host_passes) *host_passes = 1;
        return BW_OK;
    }
    if (cb < bw::kCtaBits + 1) return fail(BW_BAD_ARGUMENTS, "workspace too small: need 2^%d elements", bw::kCtaBits + 2);
    cudaStream_t st[2];
    BW_TRY(ooc_streams(dev, st));
    cudaEvent_t start;
    BW_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    BW_CUDA(cudaEventRecord(start, caller));  // order after the caller's prior work
    for (int i = 0; i < 2; ++i) BW_CUDA(cudaStreamWaitEvent(st[i], start, 0));
    cudaEventDestroy(start);
    u64* buf[2] = {reinterpret_cast<u64*>(work_dev), reinterpret_cast<u64*>(work_dev) + (1ull << cb)};
    int passes = 0;
    // Pass 0: contiguous chunks, stages 0..cb-1.
    {
        const uint64_t chunks = 1ull << (log2n - cb);
        const size_t bytes = (size_t)8 << cb;
        for (uint64_t c = 0; c < chunks; ++c) {
            const int b = (int)(c & 1);
            int64_t* h = host + (c << cb);
            BW_CUDA(cudaMemcpyAsync(buf[b], h, bytes, cudaMemcpyHostToDevice, st[b]));
            BW_TRY(fwht_impl(reinterpret_cast<int64_t*>(buf[b]), cb, nullptr, false, st[b]));
            BW_CUDA(cudaMemcpyAsync(h, buf[b], bytes, cudaMemcpyDeviceToHost, st[b]));
        }
        ++passes;
    }
    // Passes over the high bits: 2^g rows at stride 2^k x 2^13 columns.
    const int cols = bw::kCtaBits;
    const int gmax = cb - cols;
    for (int k = cb; k < log2n;) {
        {  // this pass reads what both streams wrote in the previous one: join them
            cudaEvent_t ev[2];
            for (int i = 0; i < 2; ++i) {
                BW_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
                BW_CUDA(cudaEventRecord(ev[i], st[i]));
            }
            BW_CUDA(cudaStreamWaitEvent(st[1], ev[0], 0));
            BW_CUDA(cudaStreamWaitEvent(st[0], ev[1], 0));
            for (int i = 0; i < 2; ++i) cudaEventDestroy(ev[i]);
        }
        const int rem = log2n - k;
        const int npass = (rem + gmax - 1) / gmax;
        const int g = (rem + npass - 1) / npass;
        const int w = cb - g;                                   // row width: as many columns as fit
        const uint64_t lo_chunks = 1ull << (k - w);             // bits [w, k)
        const uint64_t hi_chunks = 1ull << (log2n - k - g);     // bits [k+g, n)
        const size_t width = (size_t)8 << w, pitch = (size_t)8 << k;
        uint64_t c = 0;
        for (uint64_t hc = 0; hc < hi_chunks; ++hc)
            for (uint64_t lc = 0; lc < lo_chunks; ++lc, ++c) {
                const int b = (int)(c & 1);
                int64_t* h = host + ((lc << w) | (hc << (k + g)));
                BW_CUDA(cudaMemcpy2DAsync(buf[b], width, h, pitch, width, (size_t)1 << g, cudaMemcpyHostToDevice, st[b]));
                BW_TRY(fwht_high_bits(buf[b], cb, w, st[b]));
                BW_CUDA(cudaMemcpy2DAsync(h, pitch, buf[b], width, width, (size_t)1 << g, cudaMemcpyDeviceToHost, st[b]));
            }
        k += g;
        ++passes;
    }
    BW_CUDA(cudaStreamSynchronize(st[0]));
    BW_CUDA(cudaStreamSynchronize(st[1]));
    if (host_passes) *host_passes = passes;
    return BW_OK;
}

// inverse_wht_inplace (core.py:147-173), int64 payload.
int bw_inverse_i64(int64_t* data, int log2n, int64_t* scratch_dev, void* stream) {
    BW_TRY(check_signal(data, log2n));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    BW_TRY(bound_impl(data, log2n, scratch_dev, dev, s, nullptr));
    if (log2n == 0) return BW_OK;
    BW_TRY(fwht_impl(data, log2n, nullptr, false, s));
    void* p = nullptr;
    BW_TRY(scratch(dev, 64, &p));
    int* flag = reinterpret_cast<int*>(reinterpret_cast<char*>(p) + 32);
    BW_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    const uint64_t count = 1ull << log2n;
    const unsigned grid = (unsigned)((count + (1ull << bw::kMinmaxChunkBits) - 1) >> bw::kMinmaxChunkBits);
    bw::k_check_divisible<<<grid, 512, 0, s>>>(reinterpret_cast<const long long*>(data), count, log2n, flag);
    BW_LAUNCHED("k_check_divisible launch");
    int h = 0;
    BW_CUDA(cudaMemcpyAsync(&h, flag, sizeof h, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (h) {
        // Undo (core.py:160-166): H(Hx) = 2^n x, and 2^n divides exactly.
        BW_TRY(fwht_impl(data, log2n, nullptr, false, s));
    }
    bw::k_shift_right<<<grid, 512, 0, s>>>(reinterpret_cast<long long*>(data), count, log2n);
    BW_LAUNCHED("k_shift_right launch");
    if (h) {
        BW_CUDA(cudaStreamSynchronize(s));
        return fail(BW_INEXACT_DIVISION, "coefficients are not all divisible by 2**%d", log2n);
    }
    return BW_OK;
}

// wht_bruteforce (core.py:128-144): out of place, n <= limit (default 14).
int bw_wht_bruteforce_i64(const int64_t* x, int64_t* y, int log2n, void* stream) {
    BW_TRY(check_signal(x, log2n));
    BW_TRY(check_signal(y, log2n));
    if (log2n > 20) return fail(BW_BAD_ARGUMENTS, "brute force is O(4^n); n = %d is too large", log2n);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    const uint32_t N = 1u << log2n;
    bw::k_bruteforce<<<(N + 255) / 256, 256, 0, as_stream(stream)>>>(reinterpret_cast<const long long*>(x),
                                                                       reinterpret_cast<long long*>(y), log2n);
    BW_LAUNCHED("k_bruteforce launch");
    return BW_OK;
}

// parseval_energy partial sums (core.py:176-185): writes nblocks x (lo, hi,
// top) 64-bit words of the exact sum of squares; the caller adds them.
int bw_sumsq_partials_i64(const int64_t* x, uint64_t count, uint64_t* partial_dev, int nblocks, void* stream) {
    if (!x || !partial_dev || nblocks < 1 || count == 0) return fail(BW_BAD_ARGUMENTS, "bad arguments");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    bw::k_sumsq<<<nblocks, 256, 0, as_stream(stream)>>>(reinterpret_cast<const long long*>(x), count,
                                                        reinterpret_cast<unsigned long long*>(partial_dev));
    BW_LAUNCHED("k_sumsq launch");
    return BW_OK;
}

// fold (subspace.py:150-161) of a device signal, or of a generated one.
// GF(2) helpers of the block fold (vectors as bit masks).
namespace gf2 {
// Insert v into a reduced basis (pivot = highest set bit); returns false if
// v is dependent.  comb tracks which original vectors XOR to each basis vector.
struct Basis {
    std::vector<uint64_t> vec, comb;
    bool insert(uint64_t v, uint64_t c, uint64_t* rest_comb = nullptr) {
        for (size_t i = 0; i < vec.size(); ++i)
            if ((v ^ vec[i]) < v) {  // vec[i]'s pivot bit is set in v
                v ^= vec[i];
                c ^= comb[i];
            }
        if (v == 0) {
            if (rest_comb) *rest_comb = c;
            return false;
        }
        // keep the basis sorted by decreasing pivot so one sweep reduces
        size_t pos = 0;
        while (pos < vec.size() && vec[pos] > v) ++pos;
        vec.insert(vec.begin() + pos, v);
        comb.insert(comb.begin() + pos, c);
        return true;
    }
};
// Inverse of the d x d matrix given by its columns (invertible).
std::vector<uint64_t> inverse_cols(const std::vector<uint64_t>& col, int d) {
    // rows of [M | I]
    std::vector<uint64_t> row(d, 0), inv(d, 0);
    for (int r = 0; r < d; ++r) {
        for (int c = 0; c < d; ++c) row[r] |= ((col[c] >> r) & 1ull) << c;
        inv[r] = 1ull << r;
    }
    for (int c = 0; c < d; ++c) {
        int p = c;
        while (p < d && !((row[p] >> c) & 1)) ++p;
        std::swap(row[c], row[p]);
        std::swap(inv[c], inv[p]);
        for (int r = 0; r < d; ++r)
            if (r != c && ((row[r] >> c) & 1)) {
                row[r] ^= row[c];
                inv[r] ^= inv[c];
            }
    }
    std::vector<uint64_t> out(d, 0);  // columns of the inverse
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) out[c] |= ((inv[r] >> c) & 1ull) << r;
    return out;
}
uint64_t apply_cols(const std::vector<uint64_t>& col, uint64_t v) {
    uint64_t o = 0;
    for (size_t i = 0; i < col.size(); ++i)
        if ((v >> i) & 1) o ^= col[i];
    return o;
}
}  // namespace gf2

// Plan of the block fold (k_fold_blocks) for d_out > kFoldBlockBits.  When
// the low kFoldBlockBits columns of L are dependent, points of one chunk can
// share a bin: the plan then carries the chunk's bin table (gtab) and the
// kernel accumulates with shared-memory atomics (inj = false).
struct FoldBlockPlan {
    std::vector<uint64_t> h0;
    std::vector<unsigned> bval;
    std::vector<unsigned long long> kap;
    std::vector<unsigned> ftop, bmap, gtab;  // gtab: in-block bin of chunk point e (dependent low columns)
    uint64_t nchunk = 0;
    bool inj = true;  // the low K columns of L are independent
};

static bool fold_block_plan(const uint64_t* cols, int d_in, int d_out, FoldBlockPlan* fp) {
    constexpr int K = bw::kFoldBlockBits;
    if (d_out < 8 || d_in <= K || d_in - K > 32 || d_out > 30) return false;
    // B = [the independent low columns (of 0..K-1) | unit vectors completing a
    // basis]; A = B^-1 maps every low column into the first K coordinates
    gf2::Basis low;
    std::vector<uint64_t> B;
    for (int i = 0; i < K; ++i)
        if (low.insert(cols[i], 0)) B.push_back(cols[i]);
    fp->inj = (int)B.size() == K;
    for (int r = 0; r < d_out && (int)B.size() < d_out; ++r)
        if (low.insert(1ull << r, 0)) B.push_back(1ull << r);
    if ((int)B.size() != d_out) return false;
    const std::vector<uint64_t> A = gf2::inverse_cols(B, d_out);
    fp->gtab.clear();
    // Shared-memory atomics (no barrier per chunk) measured faster than the
    // race-free plain adds even when the chunk is injective: 2^32 -> 2^20 in
    // 5.4 vs 6.8 ms (profiles/r01_fold_atomic_ab.log).  BW_FOLD_PLAIN=1 keeps
    // the plain adds where they are race-free (A/B knob).
    if (!(getenv("BW_FOLD_PLAIN") && getenv("BW_FOLD_PLAIN")[0] == '1')) fp->inj = false;
    if (!fp->inj) {
        std::vector<uint64_t> g(K);
        for (int i = 0; i < K; ++i) {
            g[i] = gf2::apply_cols(A, cols[i]);
            if (g[i] >> K) return false;  // (cannot happen: spans of the independent low columns)
        }
        fp->gtab.assign((size_t)1 << K, 0u);
        for (uint32_t e = 1; e < (1u << K); ++e) {
            const int lowbit = __builtin_ctz(e);
            fp->gtab[e] = fp->gtab[e & (e - 1)] ^ (unsigned)g[lowbit];
        }
    }
    const int M = d_in - K;
    std::vector<uint64_t> ftop(M), fbot(M);
    for (int m = 0; m < M; ++m) {
        const uint64_t f = gf2::apply_cols(A, cols[K + m]);
        ftop[m] = f & ((1ull << K) - 1ull);
        fbot[m] = f >> K;
    }
    gf2::Basis img;
    std::vector<uint64_t> kern;
    for (int m = 0; m < M; ++m) {
        uint64_t kc = 0;
        if (!img.insert(fbot[m], 1ull << m, &kc)) kern.push_back(kc);
    }
    const int r = (int)img.vec.size(), dk = (int)kern.size();
    if (dk > 32) return false;
    fp->h0.clear();
    fp->bval.clear();
    for (uint64_t sel = 0; sel < (1ull << r); ++sel) {  // every block of the image, with a chunk on it
        uint64_t b = 0, h = 0;
        for (int i = 0; i < r; ++i)
            if ((sel >> i) & 1) {
                b ^= img.vec[i];
                h ^= img.comb[i];
            }
        fp->bval.push_back((unsigned)b);
        fp->h0.push_back(h);
    }
    fp->kap.assign(1024, 0);
    fp->ftop.assign(1024, 0);
    fp->bmap.assign(1024, 0);
    for (int g = 0; g < 4; ++g)
        for (int v = 0; v < 256; ++v)
            for (int i = 0; i < 8; ++i) {
                if (!((v >> i) & 1)) continue;
                const int bit = 8 * g + i;
                if (bit < dk) fp->kap[256 * g + v] ^= kern[bit];
                if (bit < M) fp->ftop[256 * g + v] ^= (unsigned)ftop[bit];
                if (bit < d_out) fp->bmap[256 * g + v] ^= (unsigned)B[bit];
            }
    fp->nchunk = 1ull << dk;
    return true;
}

static int fold_impl(const int64_t* x, int d_in, const uint64_t* col_masks, int d_out, int64_t* out_dev,
                     const bw::GenParams& g, cudaStream_t s) {
    if (!col_masks || !out_dev) return fail(BW_BAD_ARGUMENTS, "null pointer");
    if (d_out < 1 || d_in < d_out || d_in > 8 * bw::kFoldGroups || d_out > 30)
        return fail(BW_BAD_ARGUMENTS, "need 1 <= d_out <= d_in <= 40, d_out <= 30 (got %d, %d)", d_out, d_in);
    int dev = 0;
    BW_TRY(device_setup(&dev));
    const int groups = (d_in + 7) / 8;
    std::vector<unsigned> tab((size_t)groups * 256, 0u);
    for (int q = 0; q < groups; ++q)
        for (int v = 0; v < 256; ++v) {
            uint64_t t = 0;
            for (int b = 0; b < 8; ++b)
                if (((v >> b) & 1) && 8 * q + b < d_in) t ^= col_masks[8 * q + b];
            if (t >> d_out) return fail(BW_BAD_ARGUMENTS, "column mask wider than d_out bits");
            tab[(size_t)q * 256 + v] = (unsigned)t;
        }
    void* sc = nullptr;
    BW_TRY(scratch(dev, 4096 + tab.size() * 4, &sc));
    unsigned* dtab = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(sc) + 4096);
    BW_CUDA(cudaMemcpyAsync(dtab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, s));
    BW_CUDA(cudaMemsetAsync(out_dev, 0, (size_t)8 << d_out, s));
    const uint64_t count = 1ull << d_in;
    const int grid = grid_for(dev, count, 256, 8);
    unsigned long long* out = reinterpret_cast<unsigned long long*>(out_dev);
    FoldBlockPlan fp;
    if (fold_blocks_enabled() && fold_block_plan(col_masks, d_in, d_out, &fp)) {
        const int nb = (int)fp.bval.size();
        int nsplit = (8 * g_num_sms[dev] + nb - 1) / nb;  // ~8 CTAs per SM over the run
        if (nb == 1) nsplit = 4 * g_num_sms[dev];  // one block (d_out <= 12): one wave, fewer flush atomics
        if ((uint64_t)nsplit > fp.nchunk) nsplit = (int)fp.nchunk;
        if (nsplit < 1) nsplit = 1;
        const size_t tb = 8 * fp.h0.size() + 4 * fp.bval.size() + 8 * 1024 + 4 * 1024 * 2 + 4 * fp.gtab.size();
        void* sc2 = nullptr;
        BW_TRY(scratch(dev, 4096 + tab.size() * 4 + tb + 64, &sc2));
        char* q = reinterpret_cast<char*>(sc2) + 4096 + ((tab.size() * 4 + 15) & ~size_t(15));
        unsigned long long* dh0 = reinterpret_cast<unsigned long long*>(q);
        unsigned long long* dkap = dh0 + fp.h0.size();
        unsigned* dftop = reinterpret_cast<unsigned*>(dkap + 1024);
        unsigned* dbmap = dftop + 1024;
        unsigned* dbval = dbmap + 1024;
        BW_CUDA(cudaMemcpyAsync(dh0, fp.h0.data(), 8 * fp.h0.size(), cudaMemcpyHostToDevice, s));
        BW_CUDA(cudaMemcpyAsync(dkap, fp.kap.data(), 8 * 1024, cudaMemcpyHostToDevice, s));
        BW_CUDA(cudaMemcpyAsync(dftop, fp.ftop.data(), 4 * 1024, cudaMemcpyHostToDevice, s));
        BW_CUDA(cudaMemcpyAsync(dbmap, fp.bmap.data(), 4 * 1024, cudaMemcpyHostToDevice, s));
        BW_CUDA(cudaMemcpyAsync(dbval, fp.bval.data(), 4 * fp.bval.size(), cudaMemcpyHostToDevice, s));
        unsigned* dgtab = dbval + fp.bval.size();
        if (!fp.inj) BW_CUDA(cudaMemcpyAsync(dgtab, fp.gtab.data(), 4 * fp.gtab.size(), cudaMemcpyHostToDevice, s));
        bw::FoldBlockArgs fa;
        fa.x = reinterpret_cast<const long long*>(x);
        fa.g = g;
        fa.out = out;
        fa.h0 = dh0;
        fa.bval = dbval;
        fa.kap = dkap;
        fa.ftop = dftop;
        fa.bmap = dbmap;
        fa.gtab = dgtab;
        fa.nsplit = nsplit;
        fa.nchunk = fp.nchunk;
        constexpr size_t smem = (8 << bw::kFoldBlockBits) + 8 * 1024 + 4 * 1024 * 2;
        if (fp.inj) {
            BW_CUDA(cudaFuncSetAttribute(bw::k_fold_blocks<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            bw::k_fold_blocks<true><<<nb * nsplit, bw::kFoldThreads, smem, s>>>(fa);
        } else {
            constexpr size_t smem2 = smem + (4 << bw::kFoldBlockBits);
            BW_CUDA(cudaFuncSetAttribute(bw::k_fold_blocks<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
            bw::k_fold_blocks<false><<<nb * nsplit, bw::kFoldThreads, smem2, s>>>(fa);
        }
        BW_LAUNCHED("k_fold_blocks launch");
        BW_CUDA(cudaStreamSynchronize(s));  // the tables live in shared scratch
        return BW_OK;
    }
    if (d_out <= 14)  // up to 128 KB of shared bins: one 1024-thread CTA per SM (measured faster than 4 x 256)
        bw::k_fold<true, 1024><<<g_num_sms[dev], 1024, (size_t)8 << d_out, s>>>(
            reinterpret_cast<const long long*>(x), count, dtab, groups, d_out, out, g);
    else
        bw::k_fold<false><<<grid, 256, 0, s>>>(reinterpret_cast<const long long*>(x), count, dtab, groups, d_out, out,
                                               g);
    BW_LAUNCHED("k_fold launch");
    BW_CUDA(cudaStreamSynchronize(s));  // the table lives in shared scratch
    return BW_OK;
}

int bw_fold_i64(const int64_t* x, int d_in, const uint64_t* col_masks, int d_out, int64_t* out_dev, void* stream) {
    BW_TRY(check_signal(x, d_in));
    bw::GenParams g;
    memset(&g, 0, sizeof g);
    return fold_impl(x, d_in, col_masks, d_out, out_dev, g, as_stream(stream));
}

static int gen_params(int kind, uint64_t seed, const uint64_t* params, int nparams, bw::GenParams* g);

int bw_fold_gen_i64(int d_in, int kind, uint64_t seed, const uint64_t* params, int nparams,
                    const uint64_t* col_masks, int d_out, int64_t* out_dev, void* stream) {
    bw::GenParams g;
    BW_TRY(gen_params(kind, seed, params, nparams, &g));
    return fold_impl(nullptr, d_in, col_masks, d_out, out_dev, g, as_stream(stream));
}

// ---- multi-device plan with the cross-shard stage fused into the last pass --
//
// Local plan = low pass + high passes over n_local bits except the last r
// bits, which the fused pass (kernel K6') covers together with the log2 P
// shard bits: r + log2 P <= 10 rows of a 2-CTA tile (>= 128-byte rows).
}  // extern "C"
namespace {

// Tile of the fused pass: a 2-CTA cluster tile (2^14, 256-byte rows at the
// default r_last + log2 P = 9) when its column count fits the 2-CTA kernels
// (L = 4..8), else a single-CTA tile.
void fused_shape(int p, int r_last, int* q, int* L) {
    const int l1 = 14 - p - r_last;
    if (l1 >= 4 && l1 <= 8) {
        *q = 1;
        *L = l1;
    } else {
        *q = 0;
        *L = 13 - p - r_last;
    }
}

// Fused multi-device plan: a 13-bit low pass, local high passes, then the
// fused pass with r_last local rows + log2 P shard rows (<= 10 rows).
// r_last minimises the measured cost model (the fused pass is costed as a
// local high pass of r_last + log2 P rows at k = n_local - r_last).
int fused_plan(int nl, int p, std::vector<int>* local, int* r_last) {
    if (p < 1 || p > BW_MAX_LOG2P) return fail(BW_INVALID_WORKERS, "log2p = %d outside 1..%d", p, BW_MAX_LOG2P);
    if (nl < 14) return fail(BW_BAD_ARGUMENTS, "fused cross-shard plan needs n_local >= 14");
    long long best = -1;
    std::vector<int> hi;
    // low pass of 13, 14 or 15 bits (a 14-bit low pass saves a whole local
    // pass when n_local + log2 P = 34: 14 + 10 + (7 + 3) instead of
    // 13 + 7 + 5 + (6 + 3)), then the cheapest split, then the fused pass
    for (int w0 = 13; w0 <= 15 && w0 < nl; ++w0) {
        const int h = nl - w0;
        for (int r = 1; r <= h && r + p <= bw::kMaxHighBits; ++r) {
            int q = 0, L = 0;
            fused_shape(p, r, &q, &L);
            const int rows = r + p;
            const int eff = rows <= bw::kRegOnlyMaxBits ? shape_eff(rows, 0, nl - r) : shape_eff(rows, q, nl - r);
            const long long cost = 1000000 / kLowEff[w0 - 13] + best_high_split(w0, h - r, &hi) + 1000000 / eff;
            if (best < 0 || cost < best) {
                best = cost;
                local->assign(1, w0);
                local->insert(local->end(), hi.begin(), hi.end());
                *r_last = r;
            }
        }
    }
    if (best < 0) return fail(BW_BAD_ARGUMENTS, "no room for the fused pass");
    return BW_OK;
}


template <int LOGP, class F>
int with_fused_kernel(int L, F&& f) {
    switch (L) {
        case 3: return f(ic<3>{});
        case 4: return f(ic<4>{});
        case 5: return f(ic<5>{});
        case 6: return f(ic<6>{});
        case 7: return f(ic<7>{});
        case 8: return f(ic<8>{});
        case 9: return f(ic<9>{});
        case 10: return f(ic<10>{});
        case 11: return f(ic<11>{});
        default: return fail(BW_BAD_ARGUMENTS, "no fused kernel for %d column bits", L);
    }
}
}  // namespace
extern "C" {

int bw_plan_fused(int log2n_local, int log2p, int* widths, int* nwidths, int* r_last) {
    if (!widths || !nwidths || !r_last) return fail(BW_BAD_ARGUMENTS, "null argument");
    std::vector<int> w;
    int r = 0;
    BW_TRY(fused_plan(log2n_local, log2p, &w, &r));
    if ((int)w.size() > *nwidths) return fail(BW_BAD_ARGUMENTS, "widths array too small");
    for (size_t i = 0; i < w.size(); ++i) widths[i] = w[i];
    *nwidths = (int)w.size();
    *r_last = r;
    return BW_OK;
}

// Device `rank`'s share of the fused last pass (K6') over the P shards.
}  // extern "C"
namespace {
int xfused_pass(int64_t* const* shards, int log2p, int log2n_local, int r_last, int rank, void* stream,
                const bw::ExtractArgs* exp) {
    if (!shards || log2p < 1 || log2p > BW_MAX_LOG2P) return fail(BW_INVALID_WORKERS, "bad shard list");
    const int P = 1 << log2p;
    if (rank < 0 || rank >= P) return fail(BW_INVALID_WORKERS, "rank %d outside 0..%d", rank, P - 1);
    int q = 0, L = 0;
    fused_shape(log2p, r_last, &q, &L);
    const int TL = 13 + q - log2p;
    if (r_last < 1 || L < 3 || log2n_local < TL + log2p)
        return fail(BW_BAD_ARGUMENTS, "bad fused pass: n_local=%d r=%d p=%d", log2n_local, r_last, log2p);
    bw::ShardPtrs sp;
    memset(&sp, 0, sizeof sp);
    for (int i = 0; i < P; ++i) {
        if (!shards[i] || (reinterpret_cast<uintptr_t>(shards[i]) & 15u))
            return fail(BW_BAD_ARGUMENTS, "shard %d is null or not 16-byte aligned", i);
        sp.p[i] = reinterpret_cast<u64*>(shards[i]);
    }
    int dev = 0;
    BW_TRY(device_setup(&dev));
    const int k = log2n_local - r_last;
    const uint64_t tiles = 1ull << (log2n_local - TL), per = tiles >> log2p;
    cudaStream_t s = as_stream(stream);
    auto go = [&](auto lp) -> int {
        constexpr int LOGP = decltype(lp)::value;
        return with_fused_kernel<LOGP>(L, [&](auto l) -> int {
            constexpr int LL = decltype(l)::value;
            if (q == 1) {
                if constexpr (LL >= 4 && LL <= 8 && LL + LOGP <= 13) {
                    if (exp)
                        return launch_cfg<bw::CfgHigh14c>(bw::k_pass_x<bw::CfgHigh14c, LL, LOGP, true>,
                                                          (unsigned)(per << 1), s, sp, k, (uint64_t)rank * per, *exp,
                                                          log2n_local);
                    return launch_cfg<bw::CfgHigh14c>(bw::k_pass_x<bw::CfgHigh14c, LL, LOGP>, (unsigned)(per << 1), s,
                                                      sp, k, (uint64_t)rank * per, bw::ExtractArgs{}, log2n_local);
                }
                return fail(BW_BAD_ARGUMENTS, "no cluster fused kernel for L=%d p=%d", LL, LOGP);
            }
            if constexpr (LL + LOGP <= 12) {
                if (exp)
                    return launch_cfg<bw::CfgHigh13>(bw::k_pass_x<bw::CfgHigh13, LL, LOGP, true>, (unsigned)per, s, sp,
                                                     k, (uint64_t)rank * per, *exp, log2n_local);
                return launch_cfg<bw::CfgHigh13>(bw::k_pass_x<bw::CfgHigh13, LL, LOGP>, (unsigned)per, s, sp, k,
                                                 (uint64_t)rank * per, bw::ExtractArgs{}, log2n_local);
            } else {
                return fail(BW_BAD_ARGUMENTS, "no fused kernel for L=%d p=%d", LL, LOGP);
            }
        });
    };
    switch (log2p) {
        case 1: return go(ic<1>{});
        case 2: return go(ic<2>{});
        default: return go(ic<3>{});
    }
}
}  // namespace
extern "C" {

int bw_fwht_xfused_pass_i64(int64_t* const* shards, int log2p, int log2n_local, int r_last, int rank, void* stream) {
    return xfused_pass(shards, log2p, log2n_local, r_last, rank, stream, nullptr);
}

// The fused pass with |W| >= tau tested on its final values (configs 3/5
// over several GPUs; noisy.py:185-222): hits appended unordered with their
// global indices (base + shard * 2^n_local + offset), *count_dev accumulated.
int bw_fwht_xfused_pass_extract_i64(int64_t* const* shards, int log2p, int log2n_local, int r_last, int rank,
                                    uint64_t tau, uint64_t base, int64_t* out_idx, int64_t* out_val, uint64_t cap,
                                    uint64_t* count_dev, void* stream) {
    if (!count_dev || (cap > 0 && (!out_idx || !out_val))) return fail(BW_BAD_ARGUMENTS, "null extraction output");
    bw::ExtractArgs ex = {tau, base, reinterpret_cast<long long*>(out_idx), reinterpret_cast<long long*>(out_val),
                          reinterpret_cast<unsigned long long*>(count_dev), cap};
    return xfused_pass(shards, log2p, log2n_local, r_last, rank, stream, &ex);
}

// Cross-shard butterfly (parallel.py:103-110, all log2 P stage phases fused).
static int xshard_launch(const bw::ShardPtrs& sp, int log2p, uint64_t begin, uint64_t count, cudaStream_t s) {
    int dev = 0;
    BW_TRY(device_setup(&dev));
    if (count == 0 || log2p == 0) return BW_OK;
    const uint64_t pairs = count / 2;
    const int grid = grid_for(dev, pairs, 256, 8);
    switch (log2p) {
        case 1: bw::k_xshard<1><<<grid, 256, 0, s>>>(sp, begin, pairs); break;
        case 2: bw::k_xshard<2><<<grid, 256, 0, s>>>(sp, begin, pairs); break;
        case 3: bw::k_xshard<3><<<grid, 256, 0, s>>>(sp, begin, pairs); break;
        default: return fail(BW_INVALID_WORKERS, "log2p = %d outside 0..%d", log2p, BW_MAX_LOG2P);
    }
    BW_LAUNCHED("k_xshard launch");
    return BW_OK;
}

int bw_xshard_i64(int64_t* const* shards, int log2p, uint64_t begin, uint64_t count, void* stream) {
    if (log2p < 0 || log2p > BW_MAX_LOG2P)
        return fail(BW_INVALID_WORKERS, "log2p = %d outside 0..%d", log2p, BW_MAX_LOG2P);
    if ((begin | count) & 1ull) return fail(BW_BAD_ARGUMENTS, "begin and count must be even");
    if (!shards) return fail(BW_BAD_ARGUMENTS, "null shard list");
    bw::ShardPtrs sp;
    memset(&sp, 0, sizeof sp);
    for (int r = 0; r < (1 << log2p); ++r) {
        if (!shards[r]) return fail(BW_BAD_ARGUMENTS, "null shard %d", r);
        if (reinterpret_cast<uintptr_t>(shards[r]) & 15u)
            return fail(BW_BAD_ARGUMENTS, "shard %d is not 16-byte aligned", r);
        sp.p[r] = reinterpret_cast<u64*>(shards[r]);
    }
    return xshard_launch(sp, log2p, begin, count, as_stream(stream));
}

int bw_xshard_strided_i64(int64_t* base, uint64_t shard_stride, int log2p, uint64_t begin, uint64_t count,
                          void* stream) {
    if (!base) return fail(BW_BAD_ARGUMENTS, "null base");
    if (log2p < 0 || log2p > BW_MAX_LOG2P)
        return fail(BW_INVALID_WORKERS, "log2p = %d outside 0..%d", log2p, BW_MAX_LOG2P);
    int64_t* ptrs[8];
    for (int r = 0; r < (1 << log2p); ++r) ptrs[r] = base + r * shard_stride;
    return bw_xshard_i64(ptrs, log2p, begin, count, stream);
}

// ---- narrow-wire cross-shard stage (cross stages first, W-byte exchange) ----

// Pack a shard to wire_bytes-byte integers; *flag_dev |= 1 when some |x| >
// floor(WMAX / 2^log2p), i.e. when the narrow exchange could leave the
// wire type (the caller then runs the int64 path; the shard is unchanged).
int bw_pack_narrow_i64(const int64_t* src, uint64_t count, int wire_bytes, int log2p, void* out, uint32_t* flag_dev,
                       void* stream) {
    if (!src || !out || !flag_dev) return fail(BW_BAD_ARGUMENTS, "null pointer");
    if (wire_bytes != 1 && wire_bytes != 2) return fail(BW_BAD_ARGUMENTS, "wire is 1 or 2 bytes (got %d)", wire_bytes);
    if (log2p < 0 || log2p > BW_MAX_LOG2P)
        return fail(BW_INVALID_WORKERS, "log2p = %d outside 0..%d", log2p, BW_MAX_LOG2P);
    if (count % 8) return fail(BW_BAD_ARGUMENTS, "count must be a multiple of 8");
    if ((reinterpret_cast<uintptr_t>(src) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u))
        return fail(BW_BAD_ARGUMENTS, "source and packed buffer must be 16-byte aligned");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    if (count == 0) return BW_OK;
    const int grid = grid_for(dev, count / 8, 256, 8);
    const long long* x = reinterpret_cast<const long long*>(src);
    unsigned* f = reinterpret_cast<unsigned*>(flag_dev);
    if (wire_bytes == 1)
        bw::k_pack_narrow<signed char><<<grid, 256, 0, s>>>(x, reinterpret_cast<signed char*>(out), count,
                                                            127ll >> log2p, f);
    else
        bw::k_pack_narrow<short><<<grid, 256, 0, s>>>(x, reinterpret_cast<short*>(out), count, 32767ll >> log2p, f);
    BW_LAUNCHED("k_pack_narrow launch");
    return BW_OK;
}

// The P-point cross-shard butterfly over elements [begin, begin + count) of
// the packed shards (peer pointers); begin and count multiples of 16 / wire.
int bw_xshard_narrow(void* const* packed, int wire_bytes, int log2p, uint64_t begin, uint64_t count, void* stream) {
    if (!packed) return fail(BW_BAD_ARGUMENTS, "null shard list");
    if (wire_bytes != 1 && wire_bytes != 2) return fail(BW_BAD_ARGUMENTS, "wire is 1 or 2 bytes (got %d)", wire_bytes);
    if (log2p < 0 || log2p > BW_MAX_LOG2P)
        return fail(BW_INVALID_WORKERS, "log2p = %d outside 0..%d", log2p, BW_MAX_LOG2P);
    const uint64_t per = 16 / (uint64_t)wire_bytes;
    if ((begin | count) % per) return fail(BW_BAD_ARGUMENTS, "begin and count must be multiples of %llu", (unsigned long long)per);
    bw::NarrowPtrs sp;
    memset(&sp, 0, sizeof sp);
    for (int r = 0; r < (1 << log2p); ++r) {
        if (!packed[r] || (reinterpret_cast<uintptr_t>(packed[r]) & 15u))
            return fail(BW_BAD_ARGUMENTS, "packed shard %d is null or not 16-byte aligned", r);
        sp.p[r] = packed[r];
    }
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    if (count == 0 || log2p == 0) return BW_OK;
    const int grid = grid_for(dev, count / per, 256, 8);
    auto go = [&](auto w) -> int {
        using W = decltype(w);
        switch (log2p) {
            case 1: bw::k_xshard_narrow<W, 1><<<grid, 256, 0, s>>>(sp, begin, count); break;
            case 2: bw::k_xshard_narrow<W, 2><<<grid, 256, 0, s>>>(sp, begin, count); break;
            default: bw::k_xshard_narrow<W, 3><<<grid, 256, 0, s>>>(sp, begin, count); break;
        }
        BW_LAUNCHED("k_xshard_narrow launch");
        return BW_OK;
    };
    return wire_bytes == 1 ? go((signed char)0) : go((short)0);
}

// ---- peer memory plumbing for the one-process-per-GPU cross-shard stage ----

typedef CUresult_compat (*addr_range_fn)(unsigned long long*, size_t*, unsigned long long);

int bw_ipc_get_handle(const void* ptr, void* handle_out, uint64_t* offset_out) {
    if (!ptr || !handle_out || !offset_out) return fail(BW_BAD_ARGUMENTS, "null argument");
    // The handle names the whole allocation; the caller's pointer may sit
    // inside it (caching allocators), so report the offset from its base.
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    BW_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(BW_CUDA_ERROR, "cuMemGetAddressRange unavailable");
    unsigned long long base = 0;
    size_t size = 0;
    const int r = reinterpret_cast<addr_range_fn>(fn)(&base, &size, (unsigned long long)(uintptr_t)ptr);
    if (r != 0) return fail(BW_CUDA_ERROR, "cuMemGetAddressRange failed (%d)", r);
    cudaIpcMemHandle_t h;
    BW_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    memcpy(handle_out, &h, sizeof h);
    *offset_out = (uint64_t)((uintptr_t)ptr - base);
    return BW_OK;
}

int bw_ipc_open_handle(const void* handle, uint64_t offset, void** ptr_out) {
    if (!handle || !ptr_out) return fail(BW_BAD_ARGUMENTS, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    BW_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *ptr_out = reinterpret_cast<char*>(base) + offset;
    return BW_OK;
}

int bw_ipc_close_handle(void* ptr, uint64_t offset) {
    if (!ptr) return fail(BW_BAD_ARGUMENTS, "null argument");
    BW_CUDA(cudaIpcCloseMemHandle(reinterpret_cast<char*>(ptr) - offset));
    return BW_OK;
}

int bw_enable_peer_access(int peer_device) {
    int dev = 0;
    BW_CUDA(cudaGetDevice(&dev));
    if (dev == peer_device) return BW_OK;
    int can = 0;
    BW_CUDA(cudaDeviceCanAccessPeer(&can, dev, peer_device));
    if (!can) return fail(BW_NOT_SUPPORTED, "device %d cannot access peer %d", dev, peer_device);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return BW_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    return BW_OK;
}

static int gen_params(int kind, uint64_t seed, const uint64_t* params, int nparams, bw::GenParams* g) {
    memset(g, 0, sizeof *g);
    g->kind = kind;
    g->seed = seed;
    switch (kind) {
        case BW_GEN_PM1:
            return BW_OK;
        case BW_GEN_UNIFORM:
            if (nparams < 1 || !params) return fail(BW_BAD_ARGUMENTS, "UNIFORM needs params[0] = A");
            if (params[0] > (1ull << 62)) return fail(BW_BAD_ARGUMENTS, "A too large");
            g->a = params[0];
            return BW_OK;
        case BW_GEN_NOISY_MASKS: {
            if (nparams < 2 || !params) return fail(BW_BAD_ARGUMENTS, "NOISY_MASKS needs K, thr, masks, seeds");
            const uint64_t K = params[0];
            if (K < 1 || K > 8) return fail(BW_BAD_ARGUMENTS, "NOISY_MASKS needs 1 <= K <= 8");
            if ((uint64_t)nparams < 2 + 2 * K) return fail(BW_BAD_ARGUMENTS, "NOISY_MASKS needs 2+2K params");
            g->nmasks = (int)K;
            g->thr = params[1];
            for (uint64_t m = 0; m < K; ++m) {
                g->mask[m] = params[2 + m];
                g->mseed[m] = params[2 + K + m];
            }
            return BW_OK;
        }
        default:
            return fail(BW_BAD_ARGUMENTS, "unknown generator kind %d", kind);
    }
}

int bw_gen_range_i64(int64_t* data, uint64_t base, uint64_t count, int kind, uint64_t seed,
                     const uint64_t* params, int nparams, void* stream) {
    if (!data) return fail(BW_BAD_ARGUMENTS, "null output");
    bw::GenParams g;
    BW_TRY(gen_params(kind, seed, params, nparams, &g));
    int dev = 0;
    BW_TRY(device_setup(&dev));
    if (count == 0) return BW_OK;
    bw::k_gen<<<grid_for(dev, count, 256, 16), 256, 0, as_stream(stream)>>>(reinterpret_cast<long long*>(data),
                                                                              base, count, g);
    BW_LAUNCHED("k_gen launch");
    return BW_OK;
}

int bw_gen_i64(int64_t* data, int log2n, int kind, uint64_t seed, const uint64_t* params, int nparams,
               void* stream) {
    BW_TRY(check_signal(data, log2n));
    return bw_gen_range_i64(data, 0, 1ull << log2n, kind, seed, params, nparams, stream);
}

// Transform + extraction fused into the last pass (configs 3/5 of
// BASELINE.json: fwht, then all |W| >= tau sorted by index).
int bw_fwht_extract_i64(int64_t* data, int log2n, uint64_t tau, uint64_t base, int64_t* out_idx,
                        int64_t* out_val, uint64_t cap, void* stream, uint64_t* count) {
    BW_TRY(check_signal(data, log2n));
    if (cap > 0 && (!out_idx || !out_val)) return fail(BW_BAD_ARGUMENTS, "null output arrays");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    std::vector<int> w;
    BW_TRY(default_plan(log2n, &w));
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    const bool fusable = !passes.empty() && passes.back().kind != SMALL && !(reinterpret_cast<uintptr_t>(data) & 15u);
    if (!fusable) {
        BW_TRY(fwht_impl(data, log2n, nullptr, false, s));
        return bw_extract_ge_i64(data, log2n, tau, base, out_idx, out_val, cap, nullptr, stream, count);
    }
    // the hit counter lives apart from the compact plan's flag words (scratch() hands out one buffer per device)
    static thread_local unsigned long long* dcounts[64] = {};
    if (dev < 0 || dev >= 64) return fail(BW_BAD_ARGUMENTS, "device %d out of range", dev);
    if (!dcounts[dev]) BW_CUDA(cudaMalloc(&dcounts[dev], 64));
    unsigned long long* dcount = dcounts[dev];
    BW_CUDA(cudaMemsetAsync(dcount, 0, sizeof(unsigned long long), s));
    bw::ExtractArgs ex = {tau, base, reinterpret_cast<long long*>(out_idx), reinterpret_cast<long long*>(out_val),
                          dcount, cap};
    u64* d = reinterpret_cast<u64*>(data);
    // small-valued signals (the noisy +-1 sums of configs 3 / 5 at n <= 32): the compact plan with the
    // extraction in its low pass; larger values leave the buffer as it was for the int64 plan below
    int used = 0;
    if (compact_mode() != 0 && compact_default(log2n, data)) BW_TRY(compact_try(data, log2n, s, &used, &ex));
    if (!used)
        for (size_t i = 0; i < passes.size(); ++i)
            BW_TRY(launch_pass(passes[i], d, log2n, s, i + 1 == passes.size() ? &ex : nullptr));
    unsigned long long total = 0;
    BW_CUDA(cudaMemcpyAsync(&total, dcount, sizeof total, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (total <= cap && total <= 2048) {
        if (total > 1) {
            bw::k_sort_hits<<<1, 1024, 0, s>>>(reinterpret_cast<long long*>(out_idx), reinterpret_cast<long long*>(out_val),
                                             dcount);
            BW_LAUNCHED("k_sort_hits launch");
            BW_CUDA(cudaStreamSynchronize(s));
        }
        if (count) *count = total;
        return BW_OK;
    }
    // Too many hits to sort in one CTA (or more than cap): ordered two-phase
    // extraction over the transformed signal.
    return bw_extract_ge_i64(data, log2n, tau, base, out_idx, out_val, cap, nullptr, stream, count);
}

uint64_t bw_extract_scratch_bytes(int log2n) {
    if (log2n < 0 || log2n > BW_MAX_LOG2N) return 0;
    const uint64_t chunks = ((1ull << log2n) + (1ull << bw::kExtractChunkBits) - 1) >> bw::kExtractChunkBits;
    return (chunks + 1) * 8;
}

// extract_above (noisy.py:185-222) with |x| >= tau, ordered by index.
}  // extern "C"
namespace {
// count -> scan -> ordered write (kernel K5) for any hit predicate.
template <class H>
int extract_impl(const void* data, int log2n, H hit, uint64_t base, int64_t* out_idx_dev, void* out_val_dev,
                 uint64_t cap, void* scratch_dev, void* stream, uint64_t* count) {
    BW_TRY(check_signal(data, log2n));
    if (cap > 0 && (!out_idx_dev || !out_val_dev)) return fail(BW_BAD_ARGUMENTS, "null output arrays");
    int dev = 0;
    BW_TRY(device_setup(&dev));
    cudaStream_t s = as_stream(stream);
    const uint64_t n = 1ull << log2n;
    const uint64_t chunks = (n + (1ull << bw::kExtractChunkBits) - 1) >> bw::kExtractChunkBits;
    void* sc = scratch_dev;
    if (!sc) BW_TRY(scratch(dev, bw_extract_scratch_bytes(log2n), &sc));
    unsigned long long* counts = reinterpret_cast<unsigned long long*>(sc);
    const long long* d = reinterpret_cast<const long long*>(data);
    bw::k_extract_count<H><<<(unsigned)chunks, 512, 0, s>>>(d, n, hit, counts);
    BW_LAUNCHED("k_extract_count launch");
    bw::k_extract_scan<<<1, 1024, 0, s>>>(counts, chunks);
    BW_LAUNCHED("k_extract_scan launch");
    unsigned long long total = 0;
    BW_CUDA(cudaMemcpyAsync(&total, counts + chunks, sizeof total, cudaMemcpyDeviceToHost, s));
    BW_CUDA(cudaStreamSynchronize(s));
    if (total > 0 && cap > 0) {
        bw::k_extract_write<H><<<(unsigned)chunks, 512, 0, s>>>(d, n, hit, counts, counts + 1, base,
                                                               reinterpret_cast<long long*>(out_idx_dev),
                                                               reinterpret_cast<long long*>(out_val_dev), cap);
        BW_LAUNCHED("k_extract_write launch");
        BW_CUDA(cudaStreamSynchronize(s));
    }
    if (count) *count = total;
    if (total > cap)
        return fail(BW_CAPACITY, "%llu hits exceed the output capacity %llu", (unsigned long long)total,
                    (unsigned long long)cap);
    return BW_OK;
}
}  // namespace
extern "C" {

int bw_extract_ge_i64(const int64_t* data, int log2n, uint64_t tau, uint64_t base, int64_t* out_idx_dev,
                      int64_t* out_val_dev, uint64_t cap, void* scratch_dev, void* stream, uint64_t* count) {
    return extract_impl(data, log2n, bw::HitI64{tau}, base, out_idx_dev, out_val_dev, cap, scratch_dev, stream, count);
}

// float64 Walsh-domain signals (noisy.py:217-222 with a float chunk):
// |x| >= tau in double, hits in index order with their float64 values.
int bw_extract_ge_f64(const double* data, int log2n, double tau, uint64_t base, int64_t* out_idx_dev,
                      double* out_val_dev, uint64_t cap, void* scratch_dev, void* stream, uint64_t* count) {
    if (!(tau >= 0.0)) return fail(BW_BAD_ARGUMENTS, "tau must be >= 0");
    return extract_impl(data, log2n, bw::HitF64{tau}, base, out_idx_dev, out_val_dev, cap, scratch_dev, stream, count);
}

// ---- planner ---------------------------------------------------------------

int bw_plan_describe(int log2n, int log2p, char* json, size_t len) {
    if (log2n < 0 || log2p < 0 || log2p > BW_MAX_LOG2P || log2p > log2n || log2n - log2p > BW_MAX_LOG2N)
        return -fail(BW_BAD_ARGUMENTS, "bad plan request n=%d p=%d", log2n, log2p);
    const int nl = log2n - log2p;
    std::vector<int> w;
    default_plan(nl, &w);
    std::vector<Pass> passes;
    if (build_passes(nl, w, &passes) != BW_OK) return -BW_BAD_ARGUMENTS;
    std::string out;
    char buf[256];
    snprintf(buf, sizeof buf, "{\"log2n\":%d,\"log2p\":%d,\"local_log2n\":%d,\"passes\":[", log2n, log2p, nl);
    out += buf;
    for (size_t i = 0; i < passes.size(); ++i) {
        const Pass& p = passes[i];
        const char* kind = p.kind == SMALL ? "small" : p.kind == LOW ? "low" : p.kind == HIGH ? "high" : "reg";
        int threads = 256, smem = 8 << nl, cols = nl, tbits = nl, cluster = 1;
        unsigned long long grid = 1;
        if (p.kind != SMALL)
            visit_pass(p, [&](auto t, auto l) -> int {
                using C = typename decltype(t)::type;
                constexpr int L = decltype(l)::value;
                threads = bw::Dims<C>::NT;
                smem = bw::Dims<C>::SMEM_BYTES;
                cols = L;
                tbits = C::T;
                cluster = bw::Dims<C>::CLUSTER;
                grid = 1ull << (nl - bw::kCtaBits);
                return BW_OK;
            });
        snprintf(buf, sizeof buf,
                 "%s{\"kind\":\"%s\",\"k\":%d,\"r\":%d,\"split_a\":%d,\"k2\":%d,\"tile_bits\":%d,"
                 "\"cols_bits\":%d,\"threads\":%d,\"cluster\":%d,\"grid\":%llu,\"smem\":%d}",
                 i ? "," : "", kind, p.k, p.r, p.a, p.a ? p.k2 : 0, tbits, cols, threads, cluster, grid, smem);
        out += buf;
    }
    out += "],\"cross_stages\":[";
    for (int b = 0; b < log2p; ++b) {
        snprintf(buf, sizeof buf, "%s%d", b ? "," : "", nl + b);
        out += buf;
    }
    snprintf(buf, sizeof buf, "],\"hbm_bytes_per_pass\":%llu}", (unsigned long long)(16ull << nl));
    out += buf;
    if (json && len) {
        const size_t m = out.size() < len - 1 ? out.size() : len - 1;
        memcpy(json, out.data(), m);
        json[m] = 0;
    }
    return (int)out.size();
}

}  // extern "C"

// ---- static plan checker (host walk of the kernels' own address tables) ----
namespace {

// Virtual tile bits present in round RD's space (pre: 0..12; post: the
// tile minus the rank positions P).
template <class C, int RD>
constexpr uint32_t space_bits() {
    if (RD < C::XR || C::Q == 0) return (1u << bw::kCtaBits) - 1u;
    return ((1u << C::T) - 1u) & ~bw::p_mask<C>();
}

template <class C, int RD>
bool round_ok(std::string* why) {
    uint32_t seen = 0, regs = 0;
    auto add = [&](int b) {
        if (b < 0 || b >= C::T || ((seen >> b) & 1u)) return false;
        seen |= 1u << b;
        return true;
    };
    for (int i = 0; i < C::R; ++i) {
        if (!add(C::reg(RD, i))) { *why = "register bits overlap"; return false; }
        regs |= 1u << C::reg(RD, i);
    }
    for (int i = 0; i < 5; ++i) if (!add(C::lane(RD, i))) { *why = "lane bits overlap"; return false; }
    for (int i = 0; i < C::W; ++i) if (!add(C::warp(RD, i))) { *why = "warp bits overlap"; return false; }
    if (seen != space_bits<C, RD>()) { *why = "round does not cover its space"; return false; }
    if (C::stage(RD) & ~regs) { *why = "a staged bit is not a register bit"; return false; }
    if (RD + 1 == C::XR && C::Q > 0 && (bw::p_mask<C>() & ~regs)) {
        *why = "rank swap bits are not register bits before the exchange";
        return false;
    }
    // Bank check of the padded smem slots, for the round's own accesses and,
    // in the round before the exchange, for the DSMEM destinations.  8-byte
    // words: each half-warp must hit 16 distinct 8-byte bank pairs; 16-byte
    // words (vector rounds): each quarter-warp 8 distinct 16-byte quads.
    auto check = [&](auto slot_of, bool vec) -> bool {
        for (uint32_t warp = 0; warp < (1u << C::W); ++warp)
            for (int j = 0; j < bw::Dims<C>::E; j += vec ? 2 : 1) {
                const int group = vec ? 8 : 16;
                for (uint32_t g0 = 0; g0 < 32; g0 += group) {
                    uint32_t used = 0;
                    for (uint32_t l = 0; l < (uint32_t)group; ++l) {
                        const uint32_t slot = slot_of(g0 + l, warp, j);
                        if (vec && (slot & 1u)) return false;  // 16-byte alignment
                        const uint32_t bank = vec ? ((slot >> 1) & 7u) : (slot & 15u);
                        if ((used >> bank) & 1u) return false;
                        used |= 1u << bank;
                    }
                }
            }
        return true;
    };
    if (C::NR > 1) {
        const bool own = check(
            [&](uint32_t lane, uint32_t warp, int j) {
                return bw::smem_slot_c<C>(bw::to_local<C, RD>(bw::thread_part<C, RD>(lane, warp) | bw::reg_part<C, RD>(j)));
            },
            bw::vec_smem<C, RD>());
        if (!own) { *why = "smem bank conflict"; return false; }
        if constexpr (C::Q > 0 && RD + 1 == C::XR) {
            const bool xw = check(
                [&](uint32_t lane, uint32_t warp, int j) {
                    const uint32_t v = bw::thread_part<C, RD>(lane, warp) | bw::reg_part<C, RD>(j);
                    return bw::smem_slot_c<C>(bw::to_local<C, C::XR>(v & ~bw::p_mask<C>()));
                },
                bw::vec_smem<C, RD>());
            if (!xw) { *why = "DSMEM exchange bank conflict"; return false; }
        }
    }
    return true;
}

template <class C, int RD>
bool rounds_ok(std::string* why) {
    if constexpr (RD < C::NR) {
        if (!round_ok<C, RD>(why)) return false;
        return rounds_ok<C, RD + 1>(why);
    }
    return true;
}

template <class C, int RD, int L>
uint32_t all_stage_masks() {
    if constexpr (RD < C::NR) {
        return bw::stage_mask<C, RD, L>() | all_stage_masks<C, RD + 1, L>();
    }
    return 0;
}

template <class C, int L>
int check_pass(int n, int k, std::vector<uint8_t>& touched, uint32_t* stage_bits_out, uint64_t* bfly) {
    constexpr int T = C::T;
    std::string why;
    if (!rounds_ok<C, 0>(&why)) return fail(BW_BAD_ARGUMENTS, "layout: %s", why.c_str());
    // Stage coverage inside the tile: every row bit staged exactly once.
    uint32_t tile_stages = 0;
    int staged = 0;
    for (int rd = 0; rd < C::NR; ++rd) {
        uint32_t m = C::stage(rd);
        if (L < T) m &= ~((1u << L) - 1u);
        if (tile_stages & m) return fail(BW_BAD_ARGUMENTS, "tile bit staged twice");
        tile_stages |= m;
        staged += __builtin_popcount(m);
    }
    (void)staged;
    const uint32_t rows = L >= T ? (1u << T) - 1u : ((1u << T) - 1u) & ~((1u << L) - 1u);
    if (tile_stages != rows) return fail(BW_BAD_ARGUMENTS, "tile stages %x != rows %x", tile_stages, rows);
    uint32_t stage_bits = 0;  // the global bits the kernel's stage masks really cover
    for (int b = 0; b < T; ++b)
        if ((tile_stages >> b) & 1u)
            stage_bits |= 1u << (b < L ? b : __builtin_ctzll(bw::global_off<T, L, bw::SplitOf<C>::value>(1u << b, k)));
    *stage_bits_out = stage_bits;
    // Address walk over every (CTA, thread, register): the load layout, the
    // exchange destinations and the store layout must all be bijections.
    const uint64_t ctas = 1ull << (n - bw::kCtaBits);
    constexpr int NQ = 1 << C::Q;
    constexpr int LAST = C::NR - 1;
    std::fill(touched.begin(), touched.end(), 0);
    std::vector<uint8_t> xdst(C::Q > 0 ? (size_t)NQ << bw::kCtaBits : 0);
    for (uint64_t cta = 0; cta < ctas; ++cta) {
        const uint32_t rank = (uint32_t)(cta & (NQ - 1));
        const uint64_t base = bw::tile_base<T, L, bw::SplitOf<C>::value>(cta >> C::Q, k);
        if (C::Q > 0 && rank == 0) std::fill(xdst.begin(), xdst.end(), 0);
        for (uint32_t t = 0; t < (uint32_t)bw::Dims<C>::NT; ++t) {
            const uint32_t lane = t & 31u, warp = t >> 5;
            for (int j = 0; j < bw::Dims<C>::E; ++j) {
                const uint32_t vin = bw::thread_part<C, 0>(lane, warp) | bw::reg_part<C, 0>(j) | bw::rank_bits<C, 0>(rank);
                const uint32_t vout =
                    bw::thread_part<C, LAST>(lane, warp) | bw::reg_part<C, LAST>(j) | bw::rank_bits<C, LAST>(rank);
                const uint64_t gi = base + bw::global_off<T, L, bw::SplitOf<C>::value>(vin, k);
                const uint64_t go = base + bw::global_off<T, L, bw::SplitOf<C>::value>(vout, k);
                if (gi >= touched.size() || go >= touched.size())
                    return fail(BW_BAD_ARGUMENTS, "pass at k=%d reaches out of range", k);
                if (touched[gi] & 1) return fail(BW_BAD_ARGUMENTS, "pass at k=%d loads index %llu twice", k, (unsigned long long)gi);
                if (touched[go] & 2) return fail(BW_BAD_ARGUMENTS, "pass at k=%d stores index %llu twice", k, (unsigned long long)go);
                touched[gi] |= 1;
                touched[go] |= 2;
                if constexpr (C::Q > 0) {
                    constexpr int XW = C::XR - 1;  // round whose registers are exchanged
                    const uint32_t v = bw::thread_part<C, XW>(lane, warp) | bw::reg_part<C, XW>(j) | bw::rank_bits<C, XW>(rank);
                    uint32_t d = 0;
                    for (int i = 0; i < C::Q; ++i) d |= ((v >> C::P(i)) & 1u) << i;
                    const uint32_t slot = bw::to_local<C, C::XR>(v & ~bw::p_mask<C>());
                    uint8_t& x = xdst[((size_t)d << bw::kCtaBits) + slot];
                    if (x) return fail(BW_BAD_ARGUMENTS, "exchange writes a slot twice");
                    x = 1;
                }
            }
        }
    }
    for (uint8_t x : touched)
        if (x != 3) return fail(BW_BAD_ARGUMENTS, "pass at k=%d misses an element", k);
    *bfly += (uint64_t)__builtin_popcount(stage_bits) << (n - 1);
    return BW_OK;
}

// Host emulation of k_pass<C, L>: the same address tables, rounds, stage
// masks, cluster exchange and shared-memory slots, executed thread by thread
// on host memory (TEST HOOK; see bw_debug_emulate_i64).
template <bool FP>
void emu_butterfly(u64& a, u64& b) {
    if constexpr (FP) {
        double x, y;
        memcpy(&x, &a, 8);
        memcpy(&y, &b, 8);
        const double s = x + y, d = x - y;
        memcpy(&a, &s, 8);
        memcpy(&b, &d, 8);
    } else {
        const u64 x = a, y = b;
        a = x + y;
        b = x - y;
    }
}

template <class C, int L, int RD, bool FP = false>
void emu_stages(std::vector<u64>& v) {
    constexpr int E = bw::Dims<C>::E, NT = bw::Dims<C>::NT;
    constexpr uint32_t mask = bw::stage_mask<C, RD, L>();
    for (int t = 0; t < NT; ++t)
        for (int i = 0; i < C::R; ++i)
            if ((mask >> C::reg(RD, i)) & 1u)
                for (int j = 0; j < E; ++j)
                    if (!((j >> i) & 1))
                        emu_butterfly<FP>(v[(size_t)t * E + j], v[(size_t)t * E + (j | (1 << i))]);
}

template <class C, int L, int RD, bool FP = false>
void emu_rounds(std::vector<std::vector<u64>>& v, std::vector<std::vector<u64>>& sm) {
    constexpr int E = bw::Dims<C>::E, NT = bw::Dims<C>::NT, NQ = 1 << C::Q;
    if constexpr (RD < C::NR) {
        for (int q = 0; q < NQ; ++q)
            for (int t = 0; t < NT; ++t)
                for (int j = 0; j < E; ++j) {
                    const uint32_t vv = bw::thread_part<C, RD - 1>(t & 31, t >> 5) | bw::reg_part<C, RD - 1>(j);
                    if (RD == C::XR) {
                        const uint32_t full = vv | bw::rank_bits<C, RD - 1>((uint32_t)q);
                        uint32_t d = 0;
                        for (int i = 0; i < C::Q; ++i) d |= ((full >> C::P(i)) & 1u) << i;
                        sm[d][bw::smem_slot_c<C>(bw::to_local<C, RD>(full & ~bw::p_mask<C>()))] = v[q][(size_t)t * E + j];
                    } else {
                        sm[q][bw::smem_slot_c<C>(bw::to_local<C, RD - 1>(vv))] = v[q][(size_t)t * E + j];
                    }
                }
        for (int q = 0; q < NQ; ++q) {
            for (int t = 0; t < NT; ++t)
                for (int j = 0; j < E; ++j)
                    v[q][(size_t)t * E + j] =
                        sm[q][bw::smem_slot_c<C>(bw::to_local<C, RD>(bw::thread_part<C, RD>(t & 31, t >> 5) | bw::reg_part<C, RD>(j)))];
            emu_stages<C, L, RD, FP>(v[q]);
        }
        emu_rounds<C, L, RD + 1, FP>(v, sm);
    }
}

template <class C, int L, bool FP = false>
void emulate_pass(u64* data, int n, int k) {
    constexpr int T = C::T, E = bw::Dims<C>::E, NT = bw::Dims<C>::NT, NQ = 1 << C::Q;
    constexpr int LAST = C::NR - 1;
    std::vector<std::vector<u64>> v(NQ, std::vector<u64>((size_t)NT * E));
    std::vector<std::vector<u64>> sm(NQ, std::vector<u64>((size_t)bw::Dims<C>::CTA * 2));
    const uint64_t tiles = 1ull << (n - T);
    for (uint64_t b = 0; b < tiles; ++b) {
        const uint64_t base = bw::tile_base<T, L, bw::SplitOf<C>::value>(b, k);
        for (int q = 0; q < NQ; ++q) {
            for (int t = 0; t < NT; ++t)
                for (int j = 0; j < E; ++j)
                    v[q][(size_t)t * E + j] =
                        data[base + bw::global_off<T, L, bw::SplitOf<C>::value>(bw::thread_part<C, 0>(t & 31, t >> 5) | bw::reg_part<C, 0>(j) |
                                                             bw::rank_bits<C, 0>((uint32_t)q),
                                                         k)];
            emu_stages<C, L, 0, FP>(v[q]);
        }
        emu_rounds<C, L, 1, FP>(v, sm);
        for (int q = 0; q < NQ; ++q)
            for (int t = 0; t < NT; ++t)
                for (int j = 0; j < E; ++j)
                    data[base + bw::global_off<T, L, bw::SplitOf<C>::value>(bw::thread_part<C, LAST>(t & 31, t >> 5) | bw::reg_part<C, LAST>(j) |
                                                         bw::rank_bits<C, LAST>((uint32_t)q),
                                                     k)] = v[q][(size_t)t * E + j];
    }
}

}  // namespace

extern "C" int bw_plan_check(int log2n, const int* pass_bits, int npasses, uint64_t* butterflies) {
    if (log2n < 0 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "plan check supports 0 <= n <= 24");
    std::vector<int> w;
    if (pass_bits && npasses > 0) w.assign(pass_bits, pass_bits + npasses);
    else default_plan(log2n, &w);
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    uint64_t bfly = 0;
    uint32_t covered = 0;
    std::vector<uint8_t> touched((size_t)1 << log2n);
    for (const Pass& p : passes) {
        uint32_t bits = 0;
        int st = BW_OK;
        if (p.kind == SMALL) {
            bits = (1u << log2n) - 1u;
            bfly += (uint64_t)log2n << (log2n - 1);
        } else {
            st = visit_pass(p, [&](auto t, auto l) -> int {
                using C = typename decltype(t)::type;
                constexpr int L = decltype(l)::value;
                return check_pass<C, L>(log2n, p.karg(), touched, &bits, &bfly);
            });
        }
        if (st != BW_OK) return st;
        if (covered & bits) return fail(BW_BAD_ARGUMENTS, "stage applied twice");
        covered |= bits;
    }
    const uint32_t all = log2n ? (uint32_t)((1ull << log2n) - 1ull) : 0u;
    if (covered != all) return fail(BW_BAD_ARGUMENTS, "stages covered %x, expected %x", covered, all);
    if (butterflies) *butterflies = bfly;
    return BW_OK;
}

// TEST HOOK ONLY (never called by the product path): run the pass plan's
// exact address/stage/shared-memory tables on HOST memory, to check the
// kernels' layout logic without a GPU.  n <= 24.
extern "C" int bw_debug_emulate_i64(int64_t* host, int log2n, const int* pass_bits, int npasses) {
    if (!host || log2n < 0 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "emulation supports 0 <= n <= 24");
    std::vector<int> w;
    if (pass_bits && npasses > 0) w.assign(pass_bits, pass_bits + npasses);
    else default_plan(log2n, &w);
    std::vector<Pass> passes;
    BW_TRY(build_passes(log2n, w, &passes));
    u64* d = reinterpret_cast<u64*>(host);
    for (const Pass& p : passes) {
        if (p.kind == SMALL) {
            const uint64_t N = 1ull << log2n;
            for (int k = 0; k < log2n; ++k)
                for (uint64_t t = 0; t < N / 2; ++t) {
                    const uint64_t lo = ((t >> k) << (k + 1)) | (t & ((1ull << k) - 1)), hi = lo + (1ull << k);
                    const u64 a = d[lo], b = d[hi];
                    d[lo] = a + b;
                    d[hi] = a - b;
                }
            continue;
        }
        BW_TRY(visit_pass(p, [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            emulate_pass<C, L>(d, log2n, p.karg());
            return BW_OK;
        }));
    }
    return BW_OK;
}

// float64: the order in which a pass applies its stage bits (round by
// round, register index by register index).
namespace {
template <class C, int L, int RD>
void stage_order(int k, std::vector<int>* out) {
    if constexpr (RD < C::NR) {
        constexpr uint32_t m = bw::stage_mask<C, RD, L>();
        for (int i = 0; i < C::R; ++i) {
            const int b = C::reg(RD, i);
            if ((m >> b) & 1u) out->push_back(b < L ? b : k + (b - L));
        }
        stage_order<C, L, RD + 1>(k, out);
    }
}
}  // namespace

// Static checker of the float64 plan: the check_pass walk of every pass
// (bijective loads/stores, every stage once) plus strictly ascending stage
// order per element across the whole plan (bitwise numpy equality).
namespace {
int check_f64_plan(int log2n, bool vec, uint64_t* butterflies);
}
// Both low-pass layouts: the paired one (16-byte aligned data) and the
// 8-byte one (float64 views and int64 views that are only 8-byte aligned).
extern "C" int bw_plan_check_f64(int log2n, uint64_t* butterflies) {
    if (log2n < 0 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "plan check supports 0 <= n <= 24");
    BW_TRY(check_f64_plan(log2n, false, butterflies));
    return check_f64_plan(log2n, true, butterflies);
}
namespace {
int check_f64_plan(int log2n, bool vec, uint64_t* butterflies) {
    std::vector<Pass> passes;
    BW_TRY(f64_passes(log2n, &passes));
    uint64_t bfly = 0;
    uint32_t covered = 0;
    std::vector<int> order;
    std::vector<uint8_t> touched((size_t)1 << log2n);
    for (const Pass& p : passes) {
        uint32_t bits = 0;
        if (p.kind == SMALL) {
            bits = (1u << log2n) - 1u;
            bfly += (uint64_t)log2n << (log2n - 1);
            for (int k = 0; k < log2n; ++k) order.push_back(k);
        } else {
            BW_TRY(visit_pass_f64(p, [&](auto t, auto l) -> int {
                using C = typename decltype(t)::type;
                constexpr int L = decltype(l)::value;
                stage_order<C, L, 0>(p.k, &order);
                return check_pass<C, L>(log2n, p.k, touched, &bits, &bfly);
            }, vec));
        }
        if (covered & bits) return fail(BW_BAD_ARGUMENTS, "stage applied twice");
        covered |= bits;
    }
    const uint32_t all = log2n ? (uint32_t)((1ull << log2n) - 1ull) : 0u;
    if (covered != all) return fail(BW_BAD_ARGUMENTS, "stages covered %x, expected %x", covered, all);
    for (size_t i = 0; i < order.size(); ++i)
        if (order[i] != (int)i) return fail(BW_BAD_ARGUMENTS, "float64 stage %d applied at position %zu", order[i], i);
    if (butterflies) *butterflies = bfly;
    return BW_OK;
}
}  // namespace

// TEST HOOK ONLY: the float64 plan's exact tables executed on HOST memory
// with IEEE double add/sub (n <= 24).
extern "C" int bw_debug_emulate_f64(double* host, int log2n) {
    if (!host || log2n < 0 || log2n > 24) return fail(BW_BAD_ARGUMENTS, "emulation supports 0 <= n <= 24");
    std::vector<Pass> passes;
    BW_TRY(f64_passes(log2n, &passes));
    u64* d = reinterpret_cast<u64*>(host);
    for (const Pass& p : passes) {
        if (p.kind == SMALL) {
            const uint64_t N = 1ull << log2n;
            for (int k = 0; k < log2n; ++k)
                for (uint64_t t = 0; t < N / 2; ++t) {
                    const uint64_t lo = ((t >> k) << (k + 1)) | (t & ((1ull << k) - 1)), hi = lo + (1ull << k);
                    emu_butterfly<true>(d[lo], d[hi]);
                }
            continue;
        }
        BW_TRY(visit_pass_f64(p, [&](auto t, auto l) -> int {
            using C = typename decltype(t)::type;
            constexpr int L = decltype(l)::value;
            emulate_pass<C, L, true>(d, log2n, p.k);
            return BW_OK;
        }));
    }
    return BW_OK;
}

// Static checker of the fused cross-shard pass (mirror of check_disjoint /
// total_butterflies over all P devices): walks every device's tiles with
// the kernel's own address tables and verifies that each (shard, index) is
// loaded and stored exactly once and that the pass covers the stages
// [n_local - r_last, n_local) plus every shard bit.  n_local <= 24.
namespace {
template <class C, int LOGP, int L>
int check_fused(int nl, int r_last, uint64_t* bfly) {
    constexpr int T = C::T, TL = T - LOGP, P = 1 << LOGP, LAST = C::NR - 1, NQ = 1 << C::Q;
    const int k = nl - r_last;
    if (TL - L != r_last) return fail(BW_BAD_ARGUMENTS, "inconsistent fused shape");
    std::string why;
    if (!rounds_ok<C, 0>(&why)) return fail(BW_BAD_ARGUMENTS, "layout: %s", why.c_str());
    std::vector<uint8_t> touched((size_t)P << nl, 0);
    const uint64_t tiles = 1ull << (nl - TL), per = tiles >> LOGP;
    for (int dev = 0; dev < P; ++dev)
        for (uint64_t b = 0; b < per; ++b) {
            const uint64_t base = bw::tile_base<TL, L>((uint64_t)dev * per + b, k);
            for (int q = 0; q < NQ; ++q)
                for (uint32_t t = 0; t < (uint32_t)bw::Dims<C>::NT; ++t)
                    for (int j = 0; j < bw::Dims<C>::E; ++j) {
                        const uint32_t ei = bw::thread_part<C, 0>(t & 31, t >> 5) | bw::reg_part<C, 0>(j) |
                                            bw::rank_bits<C, 0>((uint32_t)q);
                        const uint32_t eo = bw::thread_part<C, LAST>(t & 31, t >> 5) | bw::reg_part<C, LAST>(j) |
                                            bw::rank_bits<C, LAST>((uint32_t)q);
                        const uint64_t gi =
                            ((uint64_t)(ei >> TL) << nl) + base + bw::global_off<TL, L>(ei & ((1u << TL) - 1u), k);
                        const uint64_t go =
                            ((uint64_t)(eo >> TL) << nl) + base + bw::global_off<TL, L>(eo & ((1u << TL) - 1u), k);
                        if (gi >= touched.size() || go >= touched.size())
                            return fail(BW_BAD_ARGUMENTS, "fused pass out of range");
                        if ((touched[gi] & 1) || (touched[go] & 2))
                            return fail(BW_BAD_ARGUMENTS, "fused pass touches an element twice");
                        touched[gi] |= 1;
                        touched[go] |= 2;
                    }
        }
    for (uint8_t x : touched)
        if (x != 3) return fail(BW_BAD_ARGUMENTS, "fused pass misses an element");
    // stages: every tile bit >= L = r_last local rows + LOGP shard bits, once
    uint32_t staged = 0;
    for (int rd = 0; rd < C::NR; ++rd) {
        const uint32_t m = C::stage(rd) & ~((1u << L) - 1u);
        if (staged & m) return fail(BW_BAD_ARGUMENTS, "fused pass stages a bit twice");
        staged |= m;
    }
    if (staged != (((1u << T) - 1u) & ~((1u << L) - 1u))) return fail(BW_BAD_ARGUMENTS, "fused pass stage coverage");
    *bfly = (uint64_t)(r_last + LOGP) << (nl + LOGP - 1);
    return BW_OK;
}
}  // namespace

extern "C" int bw_plan_check_fused(int log2n_local, int log2p, uint64_t* butterflies) {
    if (log2n_local > 24) return fail(BW_BAD_ARGUMENTS, "checker supports n_local <= 24");
    std::vector<int> w;
    int r = 0;
    BW_TRY(fused_plan(log2n_local, log2p, &w, &r));
    uint64_t local_bf = 0;
    BW_TRY(bw_plan_check(log2n_local - r, w.data(), (int)w.size(), &local_bf));  // the local passes' bits
    int q = 0, L = 0;
    fused_shape(log2p, r, &q, &L);
    uint64_t bf = 0;
    auto go = [&](auto lp) -> int {
        constexpr int LOGP = decltype(lp)::value;
        return with_fused_kernel<LOGP>(L, [&](auto l) -> int {
            constexpr int LL = decltype(l)::value;
            if (q == 1) {
                if constexpr (LL >= 4 && LL <= 8 && LL + LOGP <= 13)
                    return check_fused<bw::CfgHigh14c, LOGP, LL>(log2n_local, r, &bf);
                return fail(BW_BAD_ARGUMENTS, "no cluster fused kernel");
            }
            if constexpr (LL + LOGP <= 12) return check_fused<bw::CfgHigh13, LOGP, LL>(log2n_local, r, &bf);
            return fail(BW_BAD_ARGUMENTS, "no fused kernel");
        });
    };
    int st = log2p == 1 ? go(ic<1>{}) : log2p == 2 ? go(ic<2>{}) : go(ic<3>{});
    if (st != BW_OK) return st;
    // total over the 2^(n+p) signal: P shards x local stages + the fused pass
    const int n = log2n_local + log2p;
    const uint64_t total = ((uint64_t)(log2n_local - r) << (log2n_local - 1)) * (1u << log2p) + bf;
    if (total != (uint64_t)n << (n - 1)) return fail(BW_BAD_ARGUMENTS, "butterfly count %llu != n*2^(n-1)", (unsigned long long)total);
    if (butterflies) *butterflies = total;
    return BW_OK;
}
