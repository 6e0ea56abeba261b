// Host write bandwidth on the GPU box: 16.8 MB filled by T OpenMP threads
// with plain vs non-temporal AVX-512 stores (the floor of the D' expansion).
// gcc -O2 -fopenmp -mavx512f tools/exp/host_bw.c -o /tmp/host_bw && /tmp/host_bw
#include <immintrin.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>
static double now() { struct timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e6 + t.tv_nsec * 1e-3; }
int main() {
    const size_t n = 16777216;
    char *buf = aligned_alloc(64, n);
    for (size_t i = 0; i < n; ++i) buf[i] = 1;
    int threads[] = {1, 4, 8, 16};
    for (int ti = 0; ti < 4; ++ti) {
        omp_set_num_threads(threads[ti]);
        for (int nt = 0; nt < 2; ++nt) {
            double best = 1e30;
            for (int rep = 0; rep < 20; ++rep) {
                double t0 = now();
#pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n / 64; ++q) {
                    __m512i v = _mm512_set1_epi8((char)rep);
                    if (nt) _mm512_stream_si512((__m512i *)(buf + 64 * q), v);
                    else _mm512_store_si512((void *)(buf + 64 * q), v);
                }
                _mm_sfence();
                double t = now() - t0;
                if (t < best) best = t;
            }
            printf("threads %2d %s: %.1f us = %.1f GB/s\n", threads[ti], nt ? "NT   " : "plain", best, n / best / 1e3);
        }
    }
    return 0;
}
