/*
 * bigwht_b200.h -- C ABI of the B200-native fast Walsh-Hadamard transform.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `bigwht` (arXiv:1607.01039, pkg/src/bigwht).  Every entry point below
 * replaces one reference interface, cited as /root/reference/<file>:<line>.
 * The reference is pure Python + numpy; its "FFI" is the Python call itself,
 * so the binding a maintainer adds is the ctypes stub shown in
 * INTEGRATION.md (it is what paper_1607_01039_b200/_lib.py does).
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers are CUDA global memory
 *     (cudaMalloc / torch CUDA tensors); `stream` is a cudaStream_t passed as
 *     void* (NULL = legacy default stream).  Calls are asynchronous on that
 *     stream unless documented as synchronous.
 *   - The signal is caller-owned, 2^log2n int64 elements, C-contiguous,
 *     element i has index bit b of weight 2^b.  The transform is
 *     in place, natural (Sylvester/Hadamard) order, unnormalised:
 *         y_i = sum_j (-1)^popcount(i & j) x_j      (core.py:128-144)
 *   - int64 arithmetic wraps modulo 2^64 exactly like numpy int64 does in
 *     core.py:113-115, so results are bit-identical to the reference for every
 *     input, including inputs that violate the magnitude bound.
 *   - Return value: a bw_status.  On failure bw_last_error() (thread-local)
 *     holds a message.  Status codes map 1:1 onto the reference exception
 *     classes (errors.py:10-41) in the Python host layer.
 */
#ifndef BIGWHT_B200_H
#define BIGWHT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BW_ABI_VERSION 1

typedef enum bw_status {
    BW_OK = 0,
    BW_BAD_ARGUMENTS = 1,     /* errors.py:24  BadArguments          */
    BW_OVERFLOW_BOUND = 2,    /* errors.py:32  OverflowBoundError    */
    BW_INEXACT_DIVISION = 3,  /* errors.py:36  InexactDivision       */
    BW_INVALID_WORKERS = 4,   /* errors.py:40  InvalidWorkerCount    */
    BW_CAPACITY = 5,          /* extraction output capacity too small */
    BW_CUDA_ERROR = 6,        /* device failure (no reference class: DeviceError) */
    BW_NOT_SUPPORTED = 7      /* e.g. unsupported device architecture */
} bw_status;

/* Largest transform handled by one call on one device (2^34 int64 = 128 GiB). */
#define BW_MAX_LOG2N 34
/* Largest cross-shard radix (P = 2^BW_MAX_LOG2P devices / shards). */
#define BW_MAX_LOG2P 3

/* ---- library / error plumbing ------------------------------------------ */

/* ABI version (BW_ABI_VERSION). */
int bw_abi_version(void);

/* Message of the last failing call on this host thread ("" if none). */
const char *bw_last_error(void);

/* Compute capability of `device` as 10*major+minor, or -1. Synchronous. */
int bw_device_cc(int device);

/* ---- the hot path ------------------------------------------------------ */

/*
 * In-place FWHT of data[0 .. 2^log2n).  Replaces `fwht_array(buf) -> int`
 * (/root/reference/pkg/src/bigwht/core.py:97-117): no magnitude check (the
 * reference has none either), returns the butterfly count n*2^(n-1)
 * (core.py:117) in *butterflies (may be NULL).  Asynchronous, except for
 * the sizes bw_compact_auto() names (n = 26..34 by default), where the
 * compact plan is tried first and the call waits once for its first pass's
 * verdict (below: bw_fwht_i64_compact; bw_fwht_i64_int64plan never does).
 * Pass plan: one fused low-bits pass over stages 0..12/13/14 followed by
 * strided high-bits passes of <= 10 stages each, chosen by the measured
 * cost model, i.e. the blocked decomposition of
 * external.py:238-283 with many stages per HBM round trip.  data must be
 * 8-byte aligned; an 8- but not 16-byte aligned view runs the 8-byte-access
 * layouts (slower, same result).
 */
int bw_fwht_i64(int64_t *data, int log2n, void *stream, uint64_t *butterflies);

/*
 * Same transform with an explicit pass plan (test hook; mirrors the
 * reference's block-size-independence tests, test_external.py:120-129).
 * pass_bits[0] = stages of the low pass (13, 14 or 15 = a cluster of 1, 2
 * or 4 CTAs; n itself when n <= 12), the rest are the widths (1..10) of the
 * following high passes in ascending bit order, optionally r | (q+1) << 4
 * to force a cluster of 2^q CTAs; the widths must sum to log2n.
 * npasses = 0 with pass_bits = NULL runs the naive one-launch-per-stage
 * path (kernel K0, debugging/reference aid).
 */
int bw_fwht_i64_planned(int64_t *data, int log2n, const int *pass_bits,
                        int npasses, void *stream);

/* Stages [0, sum(pass_bits)) only (pass_bits as for bw_fwht_i64_planned, a
 * 13+ bit low pass first), applied to every contiguous 2^sum block of the
 * 2^log2n array: parallel.py:93-94's phase-0 chunk transforms, here the local
 * passes of the fused multi-device plan. */
int bw_fwht_i64_partial(int64_t *data, int log2n, const int *pass_bits, int npasses,
                        void *stream);

/*
 * Pass-level launches of the default plan (the passes of
 * external.py:238-283, one HBM round trip each; instrumentation: the benchmark
 * records a CUDA event between passes to time each kernel inside the step).
 * bw_plan_npasses returns the number of passes of bw_fwht_i64's plan;
 * running passes 0..npasses-1 in order equals one bw_fwht_i64 call.
 */
int bw_plan_npasses(int log2n);
int bw_fwht_i64_pass(int64_t *data, int log2n, int pass_index, void *stream);

/*
 * Pass-level form of bw_fwht_extract_i64 for instrumentation: pass
 * pass_index of the default plan with the |x| >= tau test fused into its
 * epilogue; hits are appended unordered (at most cap) and counted in
 * *count_dev (device, caller zeroes it).  bw_sort_hits_i64 then orders up to
 * 2048 hits by index.  Both asynchronous.
 */
int bw_fwht_i64_pass_extract(int64_t *data, int log2n, int pass_index, uint64_t tau,
                             uint64_t base, int64_t *out_idx, int64_t *out_val,
                             uint64_t cap, uint64_t *count_dev, void *stream);
int bw_sort_hits_i64(int64_t *idx, int64_t *val, const uint64_t *count_dev, void *stream);

/*
 * int32 input (the north_star's "seeded int32 inputs"), int64 output, out of
 * place: bit-identical to the reference's fwht_array(x.astype(int64))
 * (core.py:97-117; Signal rejects int32, core.py:56-59), with
 * overflow-free int64 accumulation (|x| < 2^31 and n <= 32 keep every sum
 * below 2^63).  The first pass reads the int32 source directly (4 B/point)
 * and writes dst; the others run in place on dst.  Asynchronous.
 */
int bw_fwht_widen_i32(const int32_t *src, int64_t *dst, int log2n, void *stream,
                      uint64_t *butterflies);

/*
 * Same for any narrow signed source: src_bytes = 4 (int32), 2 (int16) or 1
 * (int8), src aligned to 2*src_bytes.  The narrow-wire multi-device
 * transform uses it to widen its packed, already cross-transformed shard.
 */
int bw_fwht_widen(const void *src, int src_bytes, int64_t *dst, int log2n, void *stream,
                  uint64_t *butterflies);

/*
 * fwht_array with NARROW INTERMEDIATES (the +-1 Boolean-signal case of the
 * paper): the low pass reads int64 and writes int16, a middle pass writes
 * int32, the last pass writes int64 back in place -- 10 + 6 + 12 bytes per
 * point of HBM traffic for a three-pass plan instead of 3 x 16.  Each
 * intermediate is stored tile-major for the pass that reads it (contiguous
 * tile loads).  Exact: the int16 store is checked (every value after the
 * low pass within +-32767; over it, the signal is still untouched and the
 * int64 plan runs instead, *used_narrow = 0), and |y| <= 32767 * 2^r <
 * 2^31 for the <= 16 stages of the middle pass.  work: device buffer of
 * bw_narrow_scratch_bytes(log2n) bytes (0 = no narrow plan for this n: the
 * call then runs the int64 plan).  Synchronises the stream once (the flag).
 * Reference: fwht_array (core.py:97-117); results bit-identical.
 */
int bw_fwht_i64_narrow(int64_t *data, int log2n, void *work, uint64_t work_bytes, void *stream,
                       int *used_narrow, uint64_t *butterflies);
uint64_t bw_narrow_scratch_bytes(int log2n);
int bw_narrow_npasses(int log2n);
/* One narrow pass, asynchronous; pass 0 ORs 1 into *flag_dev on an int16 overflow. */
int bw_fwht_i64_narrow_pass(int64_t *data, int log2n, void *work, uint64_t work_bytes, int pass_index,
                            uint32_t *flag_dev, void *stream);
/* Test hook: static check of the narrow plan's layouts (16 <= n <= 24). */
int bw_plan_check_narrow(int log2n);

/*
 * fwht_array with COMPACT IN-PLACE INTERMEDIATES: for |x| <= lim(n)
 * (bw_compact_limit; 7 at n = 32, 31 at n = 30, 1 at n = 34 -- the +-1 Boolean signals
 * of the paper and any small-integer signal) the high-bit stages
 * run first with the signal stored as int32 inside its own buffer, and the
 * low-bit pass widens back to natural int64: 12 + 8 (m - 1) + 12 bytes per
 * point for m high passes instead of 16 per pass, and NO work buffer.  Exact:
 * no int32 intermediate can wrap below the limit, and int64 stages commute
 * (core.py:84-86), so the result is bit-identical to fwht_array.
 * max_abs >= 0: the caller's bound on |x| (fwht_inplace computes it first,
 * core.py:122): <= lim runs the plan asynchronously, above it the int64
 * plan.  max_abs < 0 (unknown, the fwht_array case): the first pass tests
 * every input; if any exceeds lim, no tile that saw it wrote anything, the
 * tiles that did are restored exactly and the int64 plan runs (synchronises
 * the stream once).  *used_compact: which plan ran.
 * Reference: fwht_array (core.py:97-117).
 */
int bw_fwht_i64_compact(int64_t *data, int log2n, long long max_abs, void *stream, int *used_compact,
                        uint64_t *butterflies);
/*
 * Whether bw_fwht_i64 / bw_fwht_inplace_i64 / bw_fwht_inplace_known_i64 try
 * the compact plan by themselves on a 16-byte aligned signal of 2^log2n
 * points: by default (BW_COMPACT unset or "auto") for the sizes where it
 * measured faster (n = 26..34: 21.7 vs 31.4 ms at n = 32, 103.8 vs 140.1 ms
 * at n = 34); BW_COMPACT=1: wherever a compact plan exists (n >= 22);
 * BW_COMPACT=0: never.  fwht_array then synchronises the stream once (the
 * first pass's verdict) and is otherwise unchanged: same result bit for bit,
 * the int64 plan for signals with larger values.
 */
int bw_compact_auto(int log2n);
/* fwht_array (core.py:97-117) on the int64 plan whatever the data: asynchronous,
 * never the compact plan (the A/B partner and fallback of bw_fwht_i64). */
int bw_fwht_i64_int64plan(int64_t *data, int log2n, void *stream, uint64_t *butterflies);
/* lim(n) of the compact plan (-1: none for this n), its pass count (0: none). */
long long bw_compact_limit(int log2n);
int bw_compact_npasses(int log2n);
/* Pass i of the compact plan (instrumentation): first stage bit, stage count, the
 * engine (32: the int32 register engine, 64: the int64 engine's mapped passes)
 * and algorithmic bytes per point (12 / 8 / 12); any pointer may be NULL. */
int bw_compact_pass_info(int log2n, int pass_index, int *k, int *r, int *engine, int *bytes_per_point);
/* One compact pass, asynchronous (instrumentation); checked = 1 only for pass 0:
 * tileflag_dev (2^(n-13) words, zeroed) and *abort_dev (zeroed) record the outcome. */
int bw_fwht_i64_compact_pass(int64_t *data, int log2n, int pass_index, int checked, uint32_t *tileflag_dev,
                             uint32_t *abort_dev, void *stream);
/* The compact plan's last pass (the widening low pass) with the threshold extraction of
 * extract_above (noisy.py:185-222, |W| >= tau) fused in, as bw_fwht_i64_pass_extract does for
 * the int64 plan; asynchronous; int32-engine plans only (n <= 32).  bw_fwht_extract_i64 runs
 * this by itself on signals the compact plan admits. */
int bw_fwht_i64_compact_pass_extract(int64_t *data, int log2n, uint64_t tau, uint64_t base, int64_t *out_idx,
                                     int64_t *out_val, uint64_t cap, uint64_t *count_dev, void *stream);
/* Test hook: the exact restore of the tiles a checked pass 0 wrote. */
int bw_fwht_i64_compact_restore(int64_t *data, int log2n, uint32_t *tileflag_dev, void *stream);
/* Test hook: static check of the compact plan (in place, layouts, coverage;
 * for the int32-engine passes also every round's bank conflicts), 16 <= n <= 24. */
int bw_plan_check_compact(int log2n);
/* Test hook: host emulation of the compact plan whose passes after the first
 * run on the int32 engine (n <= 32 plans), from the kernels' own tables;
 * 16 <= n <= 24, in place on host memory. */
int bw_debug_emulate_compact(int64_t *host, int log2n);

/*
 * float64 fwht_array (core.py:97-117 on a float64 Signal, core.py:56-59):
 * stages applied strictly in ascending order with the same IEEE a+b / a-b
 * as numpy, so results are bitwise identical to the reference (the order
 * matters in floating point).  Not the tuned int64 path.
 */
int bw_fwht_f64(double *data, int log2n, void *stream, uint64_t *butterflies);

/* inverse_wht_inplace for float64 (core.py:168-169): forward, then * 2^-n. */
int bw_inverse_f64(double *data, int log2n, void *stream);

/*
 * Max/min reduction for the int64 magnitude bound.  Writes
 * out_minmax_dev[0] = max(data), out_minmax_dev[1] = min(data) (device
 * memory, 2 int64).  Asynchronous.  Building block of
 * check_magnitude_bound (core.py:80-94).
 */
int bw_minmax_i64(const int64_t *data, uint64_t count, int64_t *out_minmax_dev,
                  void *stream);

/*
 * check_magnitude_bound(data, n) (core.py:80-94): synchronous.  Computes
 * M = max(max, -min) exactly and fails with BW_OVERFLOW_BOUND when
 * M * 2^log2n >= 2^63.  *max_abs (may be NULL) receives M (as uint64, so
 * |INT64_MIN| = 2^63 is representable).  scratch_dev: 2 int64 of device
 * memory (NULL = use an internal buffer private to the calling host thread).
 */
int bw_check_bound_i64(const int64_t *data, int log2n, int64_t *scratch_dev,
                       void *stream, uint64_t *max_abs);

/*
 * fwht_inplace(sig) (core.py:120-125) on the int64 payload: bound check
 * first -- raising BW_OVERFLOW_BOUND before any mutation, like core.py:122 --
 * then the transform.  Synchronises `stream` once (the bound read-back).
 */
int bw_fwht_inplace_i64(int64_t *data, int log2n, int64_t *scratch_dev,
                        void *stream, uint64_t *butterflies);

/*
 * fwht_inplace(sig) (core.py:120-125) when the caller knows a bound M >= max|x|
 * (a generator, a previous check): M * 2^log2n < 2^63 is checked on the host
 * (BW_OVERFLOW_BOUND before any launch, like core.py:122), then the
 * transform -- no reduction pass, no synchronisation.  max_abs < 0: the
 * device check of bw_fwht_inplace_i64.  A bound below the true max|x| is a
 * caller error (the arithmetic still wraps mod 2^64 exactly like numpy).
 */
int bw_fwht_inplace_known_i64(int64_t *data, int log2n, int64_t max_abs,
                              void *stream, uint64_t *butterflies);

/*
 * End-to-end transform of a HOST buffer (pinned for full PCIe speed):
 * H2D into the caller's device workspace (2^log2n int64), fused bound
 * check + transform on the device, D2H of the result.  If check_bound and the
 * bound fails, returns BW_OVERFLOW_BOUND with the host buffer untouched
 * (the "raise before mutation" contract of core.py:122).  Synchronous.
 */
int bw_fwht_host_i64(int64_t *host, int log2n, int64_t *work_dev,
                     int check_bound, void *stream, uint64_t *butterflies);

/*
 * A batch of host signals (fwht_array on each, core.py:97-117), bit-identical
 * to bw_fwht_host_i64 per signal.  The signals rotate over nwork (1-4)
 * distinct device buffers of 2^log2n int64, so signal i+1's host->device
 * copy overlaps signal i's device->host copy: PCIe runs full duplex, which
 * one signal alone cannot use.  With three buffers the next H2D never waits
 * for a D2H.  A buffer listed twice in a row is processed in order.
 * Synchronous.
 */
int bw_fwht_host_batch_i64(int64_t *const *host, int count, int log2n, int64_t *const *work,
                           int nwork, void *stream, uint64_t *butterflies);

/*
 * Out-of-core transform of a HOST array larger than the device workspace --
 * the paper's blocked external algorithm (external.py:65-283, PAPER.md
 * Fig. 3) with host memory in the role of the disk and the GPU as the
 * in-memory engine.  work_dev holds 2^log2_work int64 (>= 2^15).  Pass 0
 * transforms contiguous chunks of 2^(log2_work-1) elements; every further
 * pass transforms up to log2_work-14 high bits on chunks of 64 KiB-wide
 * rows moved with 2-D copies, double-buffered on two streams (H2D of one
 * chunk overlaps the other's compute and D2H).  *host_passes (may be NULL)
 * receives the number of passes over host memory.  host should be pinned
 * for full PCIe bandwidth.  Synchronous.
 */
int bw_fwht_host_ooc_i64(int64_t *host, int log2n, int64_t *work_dev, int log2_work,
                         void *stream, int *host_passes);

/*
 * inverse_wht_inplace (core.py:147-173) on the int64 payload: bound check,
 * forward transform, exact division by 2^n.  When some coefficient is not
 * divisible, the buffer is restored and BW_INEXACT_DIVISION returned
 * (core.py:160-167).  Synchronous.
 */
int bw_inverse_i64(int64_t *data, int log2n, int64_t *scratch_dev, void *stream);

/*
 * wht_bruteforce (core.py:128-144): y_i = sum_j (-1)^popcount(i & j) x_j by
 * the defining double sum, O(4^n), out of place (x unchanged).  The Python
 * layer enforces the reference's oracle limit (14 by default); the ABI
 * accepts n <= 20.  Asynchronous.
 */
int bw_wht_bruteforce_i64(const int64_t *x, int64_t *y, int log2n, void *stream);

/*
 * parseval_energy (core.py:176-185) building block: the exact sum of x^2
 * over x[0..count) as nblocks partial 192-bit integers, written to
 * partial_dev[3*b + {0,1,2}] = (low, middle, high) 64-bit words.  The sum of
 * all partials is the exact energy (beyond int64, as the reference's Python
 * int arithmetic).  Asynchronous.
 */
int bw_sumsq_partials_i64(const int64_t *x, uint64_t count, uint64_t *partial_dev,
                          int nblocks, void *stream);

/* ---- multi-device / sharded path (parallel.py:87-111 with m = P devices) */

/*
 * Cross-shard butterfly: the last log2p stages of a 2^(log2n_local+log2p)
 * transform whose P = 2^log2p shards (shard r = indices with top bits = r)
 * have each been transformed locally.  For every local index i in
 * [begin, begin+count) it gathers shards[r][i] for all r, applies the
 * P-point WHT (stage order ascending, parallel.py:103-110) and scatters the
 * results back in place.  shards[] are device pointers readable/writable
 * from the current device: local buffers (single-GPU emulation), CUDA-IPC /
 * peer-mapped buffers (one process per GPU over NVLink), or P receive slots
 * of an all-to-all.  Disjoint [begin,count) ranges may run concurrently on
 * different devices (the check_disjoint argument, parallel.py:114-134).
 * begin and count must be even.
 */
int bw_xshard_i64(int64_t *const *shards, int log2p, uint64_t begin,
                  uint64_t count, void *stream);

/*
 * Same exchange (parallel.py:103-110 stage phases) with the shards given as
 * one strided array: shard r starts at base + r*shard_stride elements
 * (all-to-all receive buffers and the single-device P-shard emulation).
 */
int bw_xshard_strided_i64(int64_t *base, uint64_t shard_stride, int log2p,
                          uint64_t begin, uint64_t count, void *stream);

/*
 * Narrow-wire cross-shard stage (parallel.py:103-110 stage phases run
 * FIRST; int64 stages on distinct bits commute, so the result is still
 * bit-identical).  If every |x| <= floor(WMAX / 2^log2p) (WMAX = 127 for a
 * 1-byte wire, 32767 for 2 bytes), no value of the P-point butterfly leaves
 * the wire type, so the exchange can move wire_bytes per point over NVLink
 * instead of 8:
 *   bw_pack_narrow_i64: shard -> packed copy; *flag_dev |= 1 if some |x| is
 *     too large (then use the int64 path; the shard is untouched).
 *     count % 8 == 0, 16-byte aligned buffers.  Asynchronous.
 *   bw_xshard_narrow: the P-point butterfly over elements [begin,
 *     begin+count) of the P packed shards (peer pointers), in place;
 *     begin, count multiples of 16 / wire_bytes.  Asynchronous.
 * then bw_fwht_widen(packed, wire_bytes, shard, n_local) on every device.
 */
int bw_pack_narrow_i64(const int64_t *src, uint64_t count, int wire_bytes, int log2p,
                       void *out, uint32_t *flag_dev, void *stream);
int bw_xshard_narrow(void *const *packed, int wire_bytes, int log2p, uint64_t begin,
                     uint64_t count, void *stream);

/*
 * Cross-shard stage FUSED into the last local pass (kernel K6'): the
 * run_parallel schedule of parallel.py:87-111 / 162-198 (phase 0 = each
 * shard's local transform, phases k = n-p..n-1 = the cross-shard stages)
 * with the stage phases merged into the last local HBM round trip.
 * bw_plan_fused gives the local plan (widths for bw_fwht_i64_partial on each
 * shard: the low pass and all high passes but the last) and r_last, the local
 * rows the fused pass takes together with the log2p shard bits
 * (r_last + log2p <= 10).  bw_fwht_xfused_pass_i64 then runs device `rank`'s
 * disjoint share of that pass: peer loads of its tiles from all P shards,
 * r_last local + log2p cross-shard stages, peer stores back -- compute and
 * NVLink exchange in one kernel.  Every device must have finished its local
 * passes before any device starts the fused pass (and all must finish before
 * the result is read).
 */
int bw_plan_fused(int log2n_local, int log2p, int *widths, int *nwidths, int *r_last);
int bw_fwht_xfused_pass_i64(int64_t *const *shards, int log2p, int log2n_local, int r_last,
                            int rank, void *stream);

/*
 * The same fused pass with the threshold test of extract_above
 * (noisy.py:185-222, |W| >= tau) on its final values: hits are appended
 * unordered to out_idx / out_val (global indices base + shard * 2^n_local +
 * offset, up to cap), their number accumulated in *count_dev; sort them with
 * bw_sort_hits_i64 (<= 2048) or on the host.  Asynchronous.
 */
int bw_fwht_xfused_pass_extract_i64(int64_t *const *shards, int log2p, int log2n_local, int r_last,
                                    int rank, uint64_t tau, uint64_t base, int64_t *out_idx,
                                    int64_t *out_val, uint64_t cap, uint64_t *count_dev, void *stream);

/*
 * Peer-memory plumbing for one process per GPU: export a device buffer as a
 * CUDA IPC handle (64 bytes) plus its offset inside the allocation, open a
 * peer's handle (NVLink peer access enabled lazily), close it again.
 * bw_enable_peer_access: single-process multi-GPU P2P from the current
 * device to peer_device.
 */
int bw_ipc_get_handle(const void *ptr, void *handle_out, uint64_t *offset_out);
int bw_ipc_open_handle(const void *handle, uint64_t offset, void **ptr_out);
int bw_ipc_close_handle(void *ptr, uint64_t offset);
int bw_enable_peer_access(int peer_device);

/* ---- signal tooling around the path ------------------------------------ */

/* Generator kinds (seeded, counter based, bit-reproducible by oracle/). */
enum bw_gen_kind {
    BW_GEN_PM1 = 1,          /* x_i = 1 - 2*(h(seed,i) & 1)                       */
    BW_GEN_UNIFORM = 2,      /* x_i = h(seed,i) mod (2A+1) - A, A = params[0]     */
    BW_GEN_NOISY_MASKS = 3   /* x_i = sum_k (1 - 2*(<s_k,i> xor [h(seed_k,i) < thr])) */
};

/*
 * Fill data[0..2^log2n) with a seeded synthetic signal.  params:
 *   PM1:         unused
 *   UNIFORM:     params[0] = A (values in [-A, A])
 *   NOISY_MASKS: params[0] = K (1..8 masks), params[1] = thr (noise
 *                probability * 2^64, an integer), params[2..2+K) = masks s_k,
 *                params[2+K..2+2K) = per-mask noise seeds.
 * Asynchronous.
 */
int bw_gen_i64(int64_t *data, int log2n, int kind, uint64_t seed,
               const uint64_t *params, int nparams, void *stream);

/* Global offset variant: element i of data gets the value of index base+i
 * of the 2^log2n signal (used by the sharded path). */
int bw_gen_range_i64(int64_t *data, uint64_t base, uint64_t count, int kind,
                     uint64_t seed, const uint64_t *params, int nparams,
                     void *stream);

/*
 * Threshold extraction (noisy.py:185-222): all (index, value) with
 * |value| >= tau, written sorted by ascending index to out_idx_dev /
 * out_val_dev (device arrays of `cap` entries).  *count (host) receives the
 * number of hits; if it exceeds cap, BW_CAPACITY is returned and nothing
 * beyond cap is written (call again with a larger cap).  |INT64_MIN| is
 * treated as 2^63.  Index offset `base` is added to every index (shards).
 * scratch_dev must hold bw_extract_scratch_bytes(log2n) bytes (NULL = use
 * an internal buffer private to the calling host thread).  Synchronous
 * (one small read-back).
 */
int bw_extract_ge_i64(const int64_t *data, int log2n, uint64_t tau,
                      uint64_t base, int64_t *out_idx_dev, int64_t *out_val_dev,
                      uint64_t cap, void *scratch_dev, void *stream,
                      uint64_t *count);
/* float64 Walsh-domain variant (noisy.py:217-222 on a float chunk): |x| >= tau
 * in double (NaN never hits), hits in index order with their float64 values;
 * same scratch and capacity rules. */
int bw_extract_ge_f64(const double *data, int log2n, double tau, uint64_t base,
                      int64_t *out_idx_dev, double *out_val_dev, uint64_t cap,
                      void *scratch_dev, void *stream, uint64_t *count);

uint64_t bw_extract_scratch_bytes(int log2n);

/*
 * The transform followed by the extraction (core.py:97-117 then
 * noisy.py:185-222), with the threshold test fused into the last pass's
 * epilogue (no extra read of the signal): equivalent to
 * bw_fwht_i64 then bw_extract_ge_i64 -- the BASELINE configs 3 and 5
 * workload.  Hits come back sorted by index.  Synchronous.
 */
int bw_fwht_extract_i64(int64_t *data, int log2n, uint64_t tau, uint64_t base,
                        int64_t *out_idx, int64_t *out_val, uint64_t cap,
                        void *stream, uint64_t *count);

/*
 * fold (subspace.py:150-161) on the device: out_dev[L.j] += x[j] for every
 * j < 2^d_in (wrapping int64 sums), where L.j is the XOR of col_masks[c]
 * (column c of the d_out x d_in binary map as a d_out-bit mask,
 * subspace.py:61-65) over the set bits c of j.  out_dev holds 2^d_out int64
 * and is zeroed first.  bw_fold_gen_i64 folds the seeded generator's signal
 * (bw_gen_i64 kinds) without materialising it.  d_in <= 40, d_out <= 30.
 * Synchronous.  WHT(fold(x, L)) = WHT(x)[row_space(L)] (subspace.py:1-11).
 */
int bw_fold_i64(const int64_t *x, int d_in, const uint64_t *col_masks, int d_out,
                int64_t *out_dev, void *stream);
int bw_fold_gen_i64(int d_in, int kind, uint64_t seed, const uint64_t *params, int nparams,
                    const uint64_t *col_masks, int d_out, int64_t *out_dev, void *stream);

/* ---- planner ----------------------------------------------------------- */

/*
 * Describe the pass plan for a 2^log2n transform over 2^log2p shards as JSON:
 *   {"log2n":..,"log2p":..,"local_log2n":..,"passes":[{"kind":"low"|"high"|
 *    "reg"|"small","k":..,"r":..,"tile_bits":..,"cols_bits":..,
 *    "threads":..,"grid":..,"smem":..}, ...], "cross_stages":[..],
 *    "hbm_bytes_per_pass":..}
 * Returns the needed length (excluding NUL); writes at most len bytes.
 */
int bw_plan_describe(int log2n, int log2p, char *json, size_t len);

/*
 * Static plan checker (mirror of parallel.py:114-147 check_disjoint /
 * total_butterflies for GPU pass plans): walks, on the host, exactly the
 * address tables the kernels use and verifies that within every pass each
 * element is touched by exactly one (CTA, thread, register) and that every
 * stage 0..log2n-1 is applied exactly once.  Exhaustive; log2n <= 24.
 * pass_bits as in bw_fwht_i64_planned (NULL = default plan).
 */
int bw_plan_check(int log2n, const int *pass_bits, int npasses,
                  uint64_t *butterflies);

/* Static checker of the multi-device plan with the fused cross-shard pass
 * (parallel.py:114-147 check_disjoint / total_butterflies over all devices):
 * every (shard, index) loaded and stored once per pass over all devices,
 * every stage of the 2^(n_local+log2p) transform applied once.
 * n_local <= 24. */
int bw_plan_check_fused(int log2n_local, int log2p, uint64_t *butterflies);

/* Static checker of the float64 plan: ascending stage order per element
 * (numpy's order, core.py:108-115; the float64 bit-identity of
 * test_parallel.py:123-129) on top of the bw_plan_check walk.  n <= 24. */
int bw_plan_check_f64(int log2n, uint64_t *butterflies);

/* TEST HOOK ONLY: the float64 plan's address tables run on host memory with
 * IEEE double add/sub.  n <= 24. */
int bw_debug_emulate_f64(double *host, int log2n);

/*
 * TEST HOOK ONLY -- never used by any product entry point.  Executes the
 * default (or given) pass plan's exact address, stage-mask and shared-memory
 * tables on HOST memory, so the kernels' layout logic is testable without a
 * GPU.  log2n <= 24.
 */
int bw_debug_emulate_i64(int64_t *host, int log2n, const int *pass_bits, int npasses);

#ifdef __cplusplus
}
#endif

#endif /* BIGWHT_B200_H */
