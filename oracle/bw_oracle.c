/*
 * bw_oracle.c -- CPU restatement of the reference FWHT path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * bench.py cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product.
 *
 * Each function cites the reference code it restates
 * (/root/reference/pkg/src/bigwht/<file>:<line>).  The generators restate this
 * repository's own seeded generator spec,
 * which the reference does not have.  Pinned against the reference itself via
 * the golden fixtures in tests/golden/ (see tests/test_oracle.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* core.py:97-117 fwht_array: for k = 0..n-1, pairs = buf.reshape(-1, 2, 2^k);
 * diff = lo - hi; lo += hi; hi = diff.  Arithmetic wraps mod 2^64 like numpy
 * int64 (done in uint64 to keep C well defined).  Returns n * 2^(n-1). */
uint64_t oracle_fwht_i64(int64_t *buf, int n) {
    uint64_t *x = (uint64_t *)buf;
    const uint64_t dim = 1ull << n;
    uint64_t butterflies = 0;
    for (int k = 0; k < n; ++k) {
        const uint64_t stride = 1ull << k;
        for (uint64_t base = 0; base < dim; base += 2 * stride) {
            uint64_t *lo = x + base, *hi = x + base + stride;
            for (uint64_t j = 0; j < stride; ++j) {
                const uint64_t a = lo[j], b = hi[j];
                lo[j] = a + b;
                hi[j] = a - b;
            }
            butterflies += stride;
        }
    }
    return butterflies;
}

/* float64 variant (core.py:97-117 on a float64 buffer): same stage order,
 * same IEEE operations (a - b, a + b), so results are bitwise identical. */
void oracle_fwht_f64(double *x, int n) {
    const uint64_t dim = 1ull << n;
    for (int k = 0; k < n; ++k) {
        const uint64_t stride = 1ull << k;
        for (uint64_t base = 0; base < dim; base += 2 * stride) {
            double *lo = x + base, *hi = x + base + stride;
            for (uint64_t j = 0; j < stride; ++j) {
                const double d = lo[j] - hi[j];
                lo[j] += hi[j];
                hi[j] = d;
            }
        }
    }
}

/* ---- parallel.py restatement: plan_parallel (87-111) + run_parallel
 * (162-198) with one pthread per worker and a join (= barrier) per phase. */
typedef struct {
    uint64_t *x;
    uint64_t start, stride, count; /* stage workload (parallel.py:24-43) */
    int chunk_n;                   /* >= 0: chunk WHT of 2^chunk_n at start */
} work_t;

static void *run_work(void *arg) {
    work_t *w = (work_t *)arg;
    if (w->chunk_n >= 0) {
        oracle_fwht_i64((int64_t *)(w->x + w->start), w->chunk_n); /* _run_chunk, 150-151 */
    } else {                                                         /* _run_workload, 154-159 */
        uint64_t *lo = w->x + w->start, *hi = w->x + w->start + w->stride;
        for (uint64_t j = 0; j < w->count; ++j) {
            const uint64_t a = lo[j], b = hi[j];
            lo[j] = a + b;
            hi[j] = a - b;
        }
    }
    return NULL;
}

/* Returns 0 on success, -1 for an invalid p (parallel.py:95-99). */
int oracle_run_parallel_i64(int64_t *buf, int n, int p) {
    if (p < 1 || p > n - 1) return -1;
    const int m = 1 << p;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * m);
    work_t *w = (work_t *)malloc(sizeof(work_t) * m);
    const uint64_t chunk = 1ull << (n - p);
    for (int i = 0; i < m; ++i) { /* phase 0 */
        w[i].x = (uint64_t *)buf;
        w[i].start = (uint64_t)i * chunk;
        w[i].chunk_n = n - p;
        w[i].stride = w[i].count = 0;
        pthread_create(&th[i], NULL, run_work, &w[i]);
    }
    for (int i = 0; i < m; ++i) pthread_join(th[i], NULL);
    const uint64_t count = 1ull << (n - 1 - p);
    for (int k = n - p; k < n; ++k) { /* stage phases, start formula 108 */
        for (int i = 0; i < m; ++i) {
            const uint64_t t = (uint64_t)i * count;
            w[i].x = (uint64_t *)buf;
            w[i].start = ((t >> k) << (k + 1)) | (t & ((1ull << k) - 1));
            w[i].stride = 1ull << k;
            w[i].count = count;
            w[i].chunk_n = -1;
            pthread_create(&th[i], NULL, run_work, &w[i]);
        }
        for (int i = 0; i < m; ++i) pthread_join(th[i], NULL);
    }
    free(th);
    free(w);
    return 0;
}

/* core.py:80-94 check_magnitude_bound: M = max(max, -min) (exact, unsigned);
 * returns 1 when M * 2^n >= 2^63 (overflow possible), else 0. */
int oracle_bound_violated(const int64_t *x, uint64_t count, int n, uint64_t *max_abs) {
    int64_t mx = INT64_MIN, mn = INT64_MAX;
    for (uint64_t i = 0; i < count; ++i) {
        if (x[i] > mx) mx = x[i];
        if (x[i] < mn) mn = x[i];
    }
    const uint64_t a = mx > 0 ? (uint64_t)mx : 0, b = mn < 0 ? (uint64_t)0 - (uint64_t)mn : 0;
    const uint64_t M = a > b ? a : b;
    if (max_abs) *max_abs = M;
    if (M == 0) return 0;
    if (n >= 63) return 1;
    return M >= (1ull << (63 - n));
}

/* ---- generators: restatement of the seeded counter-based spec ---------- */
static inline uint64_t fmix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
static inline uint64_t hash64(uint64_t seed, uint64_t i) { return fmix64((i * 0x9E3779B97F4A7C15ull) ^ seed); }

uint64_t oracle_hash64(uint64_t seed, uint64_t i) { return hash64(seed, i); }

typedef struct {
    int kind, nmasks;
    uint64_t seed, a, thr, mask[8], mseed[8];
} gen_t;

static int gen_setup(gen_t *g, int kind, uint64_t seed, const uint64_t *params, int nparams) {
    memset(g, 0, sizeof *g);
    g->kind = kind;
    g->seed = seed;
    if (kind == 1) return 0;
    if (kind == 2) {
        if (nparams < 1) return -1;
        g->a = params[0];
        return 0;
    }
    if (kind == 3) {
        if (nparams < 2) return -1;
        const uint64_t K = params[0];
        if (K < 1 || K > 8 || (uint64_t)nparams < 2 + 2 * K) return -1;
        g->nmasks = (int)K;
        g->thr = params[1];
        for (uint64_t m = 0; m < K; ++m) {
            g->mask[m] = params[2 + m];
            g->mseed[m] = params[2 + K + m];
        }
        return 0;
    }
    return -1;
}

static inline int64_t gen_value(const gen_t *g, uint64_t i) {
    if (g->kind == 1) return 1 - 2 * (int64_t)(hash64(g->seed, i) & 1ull);
    if (g->kind == 2) return (int64_t)(hash64(g->seed, i) % (2 * g->a + 1)) - (int64_t)g->a;
    int64_t x = 0;
    for (int m = 0; m < g->nmasks; ++m) {
        const uint64_t bit = (uint64_t)(__builtin_popcountll(g->mask[m] & i) & 1) ^ (uint64_t)(hash64(g->mseed[m], i) < g->thr);
        x += 1 - 2 * (int64_t)bit;
    }
    return x;
}

typedef struct {
    const gen_t *g;
    int64_t *out;
    uint64_t base, lo, hi;
    /* fold */
    const uint64_t *col;
    int d_in;
    int64_t *acc;
} gen_job_t;

static void *gen_worker(void *arg) {
    gen_job_t *j = (gen_job_t *)arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) j->out[i] = gen_value(j->g, j->base + i);
    return NULL;
}

int oracle_gen_i64(int64_t *out, uint64_t base, uint64_t count, int kind, uint64_t seed, const uint64_t *params,
                   int nparams, int threads) {
    gen_t g;
    if (gen_setup(&g, kind, seed, params, nparams)) return -1;
    if (threads < 1) threads = 1;
    pthread_t th[256];
    gen_job_t jobs[256];
    if (threads > 256) threads = 256;
    for (int t = 0; t < threads; ++t) {
        jobs[t].g = &g;
        jobs[t].out = out;
        jobs[t].base = base;
        jobs[t].lo = count * t / threads;
        jobs[t].hi = count * (t + 1) / threads;
        pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* ---- subspace.py restatement: fold (150-161) with L.j computed from the
 * column masks (column_masks, 62-65): L.j = XOR of col[c] over set bits c of j,
 * i.e. apply_map_array (116-121).  The generated signal is produced on the
 * fly so 2^34-point inputs never need to be materialised. */
static void *fold_worker(void *arg) {
    gen_job_t *j = (gen_job_t *)arg;
    /* table-driven L.j: 8-bit column groups */
    const int groups = (j->d_in + 7) / 8;
    uint64_t *tab = (uint64_t *)calloc((size_t)groups * 256, sizeof(uint64_t));
    for (int gi = 0; gi < groups; ++gi)
        for (int v = 0; v < 256; ++v) {
            uint64_t r = 0;
            for (int b = 0; b < 8; ++b)
                if (((v >> b) & 1) && gi * 8 + b < j->d_in) r ^= j->col[gi * 8 + b];
            tab[gi * 256 + v] = r;
        }
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        uint64_t t = 0;
        for (int gi = 0; gi < groups; ++gi) t ^= tab[gi * 256 + ((i >> (8 * gi)) & 255)];
        const int64_t v = j->g ? gen_value(j->g, i) : j->out[i];
        j->acc[t] += v;
    }
    free(tab);
    return NULL;
}

/* out[2^d_out] = fold(x, L); x = the generated signal (kind>0) or src (kind 0). */
int oracle_fold_i64(const int64_t *src, int d_in, const uint64_t *col_masks, int d_out, int kind, uint64_t seed,
                    const uint64_t *params, int nparams, int threads, int64_t *out) {
    gen_t g;
    const gen_t *gp = NULL;
    if (kind > 0) {
        if (gen_setup(&g, kind, seed, params, nparams)) return -1;
        gp = &g;
    }
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    const uint64_t dim = 1ull << d_in, dout = 1ull << d_out;
    pthread_t th[256];
    gen_job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].g = gp;
        jobs[t].out = (int64_t *)src;
        jobs[t].base = 0;
        jobs[t].lo = dim * t / threads;
        jobs[t].hi = dim * (t + 1) / threads;
        jobs[t].col = col_masks;
        jobs[t].d_in = d_in;
        jobs[t].acc = (int64_t *)calloc(dout, sizeof(int64_t));
        pthread_create(&th[t], NULL, fold_worker, &jobs[t]);
    }
    memset(out, 0, dout * sizeof(int64_t));
    for (int t = 0; t < threads; ++t) {
        pthread_join(th[t], NULL);
        for (uint64_t i = 0; i < dout; ++i) out[i] += jobs[t].acc[i];
        free(jobs[t].acc);
    }
    return 0;
}

/* noisy.py:217-222 _extract with |x| >= tau (|INT64_MIN| = 2^63); writes at
 * most cap hits in index order; returns the total number of hits. */
uint64_t oracle_extract_ge_i64(const int64_t *x, uint64_t count, uint64_t tau, int64_t *idx, int64_t *val,
                               uint64_t cap) {
    uint64_t h = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t mag = x[i] < 0 ? (uint64_t)0 - (uint64_t)x[i] : (uint64_t)x[i];
        if (mag >= tau) {
            if (h < cap) {
                idx[h] = (int64_t)i;
                val[h] = x[i];
            }
            ++h;
        }
    }
    return h;
}
