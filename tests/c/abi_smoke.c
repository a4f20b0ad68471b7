/* C-only consumer of the drop-in boundary (include/bigwht_b200.h): no Python,
 * no torch.  Allocates device memory with the CUDA runtime, transforms a
 * seeded 2^n int64 signal with bw_fwht_i64 and the fused extraction, and
 * checks both against the C oracle (oracle/bw_oracle.c, test infrastructure).
 *
 *   gcc -O2 -std=c11 -I include -I /usr/local/cuda/include tests/c/abi_smoke.c \
 *       -L paper_1607_01039_b200/lib -lbigwht_b200 -L oracle -loracle \
 *       -L /usr/local/cuda/lib64 -lcudart -o abi_smoke
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "bigwht_b200.h"

uint64_t oracle_fwht_i64(int64_t *buf, int n);
int oracle_gen_i64(int64_t *out, uint64_t base, uint64_t count, int kind, uint64_t seed, const uint64_t *params,
                   int nparams, int threads);

static int check(int st, const char *what) {
    if (st != BW_OK) {
        fprintf(stderr, "%s failed: status %d: %s\n", what, st, bw_last_error());
        exit(1);
    }
    return st;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 24;
    const uint64_t count = 1ull << n;
    const uint64_t amp = 1u << 20;
    int64_t *x = malloc(count * sizeof *x), *ref = malloc(count * sizeof *ref), *got = malloc(count * sizeof *got);
    if (!x || !ref || !got) return 2;
    if (oracle_gen_i64(x, 0, count, 2, 12345, &amp, 1, 4) != 0) return 2; /* uniform in [-2^20, 2^20] */
    memcpy(ref, x, count * sizeof *x);
    const uint64_t bf_ref = oracle_fwht_i64(ref, n);

    int64_t *d = NULL;
    if (cudaMalloc((void **)&d, count * sizeof *d) != cudaSuccess) return 2;
    cudaMemcpy(d, x, count * sizeof *x, cudaMemcpyHostToDevice);
    uint64_t bf = 0;
    check(bw_fwht_i64(d, n, NULL, &bf), "bw_fwht_i64");
    cudaMemcpy(got, d, count * sizeof *got, cudaMemcpyDeviceToHost);
    if (bf != bf_ref || memcmp(got, ref, count * sizeof *got) != 0) {
        fprintf(stderr, "transform differs from the oracle\n");
        return 1;
    }

    /* fused extraction: |W| >= tau with tau = 90% of the largest |W| (a few hits) */
    uint64_t mx = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t m = ref[i] < 0 ? (uint64_t)0 - (uint64_t)ref[i] : (uint64_t)ref[i];
        if (m > mx) mx = m;
    }
    const uint64_t tau = mx - mx / 10;
    uint64_t want = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t m = ref[i] < 0 ? (uint64_t)0 - (uint64_t)ref[i] : (uint64_t)ref[i];
        want += m >= tau;
    }
    cudaMemcpy(d, x, count * sizeof *x, cudaMemcpyHostToDevice);
    int64_t *didx = NULL, *dval = NULL;
    const uint64_t cap = 4096;
    cudaMalloc((void **)&didx, cap * sizeof *didx);
    cudaMalloc((void **)&dval, cap * sizeof *dval);
    uint64_t hits = 0;
    check(bw_fwht_extract_i64(d, n, tau, 0, didx, dval, cap, NULL, &hits), "bw_fwht_extract_i64");
    int64_t hidx[4096], hval[4096];
    cudaMemcpy(hidx, didx, hits * sizeof *hidx, cudaMemcpyDeviceToHost);
    cudaMemcpy(hval, dval, hits * sizeof *hval, cudaMemcpyDeviceToHost);
    if (hits != want) {
        fprintf(stderr, "extraction found %llu hits, oracle %llu\n", (unsigned long long)hits,
                (unsigned long long)want);
        return 1;
    }
    for (uint64_t h = 0; h < hits; ++h)
        if ((h && hidx[h] <= hidx[h - 1]) || hval[h] != ref[hidx[h]]) {
            fprintf(stderr, "extraction hit %llu wrong\n", (unsigned long long)h);
            return 1;
        }
    /* error path: a non-power-of-two request is refused with a message */
    if (bw_fwht_i64(NULL, n, NULL, NULL) != BW_BAD_ARGUMENTS || !bw_last_error()[0]) return 1;
    printf("c abi ok n=%d butterflies=%llu hits=%llu\n", n, (unsigned long long)bf, (unsigned long long)hits);
    cudaFree(d);
    cudaFree(didx);
    cudaFree(dval);
    free(x);
    free(ref);
    free(got);
    return 0;
}
