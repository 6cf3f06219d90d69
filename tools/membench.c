/* membench.c -- engine-free host DRAM read bandwidth (bench.py's host_dram.peak).
 *
 * Measures what the box's host memory delivers to all cores, with NO Eq. 5 arithmetic, on
 * the same memory the value store lives in (pinned, registered), so the heterogeneous
 * split's host share (§3.2 "CPU part") is judged against the hardware
 * rather than against our own engine:
 *   hm_random_rows: every thread reads `row_bytes`-byte rows at uniformly random row offsets
 *                   (xorshift64*), `batch` rows prefetched before they are read (the memory-
 *                   level parallelism a row gather can have), each row summed as uint64 words
 *                   so the loads cannot be elided;
 *   hm_sorted_rows: the Eq. 5 access SHAPE without its arithmetic: every thread walks its
 *                   contiguous slice keeping each row with probability 1/stride (a sorted
 *                   random subset, like a kept list at density 1/stride), 16 rows prefetched
 *                   ahead, row words summed;
 *   hm_sequential:  every thread streams its contiguous slice once (uint64 sums, 8 streams,
 *                   software prefetch 1 KiB ahead).
 * Returns GB/s (1e9 B/s) of bytes read; `sink` receives the checksum.
 * Build: gcc -O2 -fopenmp -march=native -shared -fPIC -o libmembench.so membench.c */
#include <omp.h>
#include <stdint.h>
#include <string.h>
#include <time.h>

static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static inline uint64_t xs64(uint64_t *s)
{
    uint64_t x = *s;
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    *s = x;
    return x * 0x2545F4914F6CDD1Dull;
}

double hm_random_rows(const void *buf, uint64_t bytes, uint64_t row_bytes, uint64_t rows_per_thread,
                      int threads, int batch, uint64_t *sink)
{
    if (!buf || row_bytes < 64 || row_bytes % 64 || bytes < row_bytes || threads < 1) return -1.0;
    if (batch < 1) batch = 1;
    if (batch > 64) batch = 64;
    const uint64_t nrows = bytes / row_bytes;
    const uint64_t words = row_bytes / 8;
    uint64_t total = 0;
    double t0 = 0, t1 = 0;
#pragma omp parallel num_threads(threads) reduction(+ : total)
    {
        uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(omp_get_thread_num() + 1);
        uint64_t acc = 0;
        const char *base = (const char *)buf;
        const char *rows[64];
#pragma omp barrier
#pragma omp master
        t0 = now_s();
#pragma omp barrier
        for (uint64_t r = 0; r < rows_per_thread; r += (uint64_t)batch) {
            for (int b = 0; b < batch; ++b) {
                rows[b] = base + (uint64_t)(((unsigned __int128)xs64(&s) * nrows) >> 64) * row_bytes;
                for (uint64_t o = 0; o < row_bytes; o += 64) __builtin_prefetch(rows[b] + o, 0, 0);
            }
            for (int b = 0; b < batch; ++b) {
                const uint64_t *w = (const uint64_t *)rows[b];
                for (uint64_t k = 0; k < words; ++k) acc += w[k];
            }
        }
#pragma omp barrier
#pragma omp master
        t1 = now_s();
        total += acc;
    }
    if (sink) *sink = total;
    const double rows_read = (double)((rows_per_thread + batch - 1) / batch * batch) * threads;
    return rows_read * (double)row_bytes / (t1 - t0) / 1e9;
}

double hm_sorted_rows(const void *buf, uint64_t bytes, uint64_t row_bytes, uint32_t stride, int threads,
                      uint64_t *sink)
{
    if (!buf || row_bytes < 64 || row_bytes % 64 || bytes < row_bytes || threads < 1 || stride < 1) return -1.0;
    const uint64_t nrows = bytes / row_bytes, words = row_bytes / 8;
    uint64_t total = 0, kept = 0;
    double t0 = 0, t1 = 0;
#pragma omp parallel num_threads(threads) reduction(+ : total, kept)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const uint64_t lo = nrows * (uint64_t)t / (uint64_t)nt, hi = nrows * (uint64_t)(t + 1) / (uint64_t)nt;
        uint64_t s = 0x9E3779B97F4A7C15ull * (uint64_t)(t + 1), acc = 0, nk = 0;
        const char *base = (const char *)buf;
        uint64_t ring[16];
        int head = 0, fill = 0;
#pragma omp barrier
#pragma omp master
        t0 = now_s();
#pragma omp barrier
        for (uint64_t r = lo; r < hi; ++r) {
            if ((uint32_t)(xs64(&s) >> 32) % stride) continue;
            const char *p = base + r * row_bytes;
            for (uint64_t o = 0; o < row_bytes; o += 64) __builtin_prefetch(p + o, 0, 0);
            if (fill == 16) {  /* consume the row prefetched 16 kept rows ago */
                const uint64_t *w = (const uint64_t *)(base + ring[head] * row_bytes);
                for (uint64_t k = 0; k < words; ++k) acc += w[k];
                ++nk;
            } else {
                ++fill;
            }
            ring[head] = r;
            head = (head + 1) & 15;
        }
        for (int i = 0; i < fill; ++i) {
            const uint64_t *w = (const uint64_t *)(base + ring[(head + i) & 15] * row_bytes);
            for (uint64_t k = 0; k < words; ++k) acc += w[k];
            ++nk;
        }
#pragma omp barrier
#pragma omp master
        t1 = now_s();
        total += acc;
        kept += nk;
    }
    if (sink) *sink = total;
    return (double)kept * (double)row_bytes / (t1 - t0) / 1e9;
}

double hm_sequential(const void *buf, uint64_t bytes, int threads, uint64_t *sink)
{
    if (!buf || bytes < 4096 || threads < 1) return -1.0;
    const uint64_t words = bytes / 8;
    uint64_t total = 0;
    double t0 = 0, t1 = 0;
#pragma omp parallel num_threads(threads) reduction(+ : total)
    {
        const int t = omp_get_thread_num(), nt = omp_get_num_threads();
        const uint64_t lo = words * (uint64_t)t / (uint64_t)nt, hi = words * (uint64_t)(t + 1) / (uint64_t)nt;
        const uint64_t *w = (const uint64_t *)buf;
        uint64_t a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma omp barrier
#pragma omp master
        t0 = now_s();
#pragma omp barrier
        uint64_t k = lo;
        for (; k + 8 <= hi; k += 8) {
            __builtin_prefetch(w + k + 128, 0, 0);
            for (int u = 0; u < 8; ++u) a[u] += w[k + u];
        }
        for (; k < hi; ++k) a[0] += w[k];
#pragma omp barrier
#pragma omp master
        t1 = now_s();
        for (int u = 0; u < 8; ++u) total += a[u];
    }
    if (sink) *sink = total;
    return (double)(words * 8) / (t1 - t0) / 1e9;
}
