/*
 * fill.c -- the seeded_inputs byte stream in C (no finite-field arithmetic),
 * multithreaded, for host-side regeneration of full-size inputs (C3: 6.3 GB,
 * C4: 32 GiB, C5: 128 GiB of sources per field) that the numpy definition in
 * seeded_inputs/__init__.py produces at ~0.1 GB/s.  Same definition:
 *
 *   key(seed, stream) = seed ^ (stream * 0xD1B54A32D192ED03)
 *   word(w)           = mix64(key + (w + 1) * 0x9E3779B97F4A7C15)
 *   byte(j)           = (word(j >> 3) >> (8 * (j & 7))) & 0xFF
 *
 * with mix64 the splitmix64 finaliser.  tests/test_inputs.py pins this file
 * byte-equal to the numpy definition.  Test infrastructure only.
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* dst[r * cols + c] = byte(base + r * row_stride + c) & mask */
static void fill_rows(uint8_t *dst, size_t r0, size_t r1, size_t cols, uint64_t key, uint64_t base,
                      uint64_t row_stride, uint8_t mask)
{
    const uint64_t gamma = 0x9E3779B97F4A7C15ull;
    for (size_t r = r0; r < r1; r++) {
        uint8_t *out = dst + r * cols;
        uint64_t j = base + r * row_stride;
        size_t c = 0;
        while (c < cols && (j & 7)) {                       /* head: partial word */
            out[c++] = (uint8_t)(mix64(key + ((j >> 3) + 1) * gamma) >> (8 * (j & 7))) & mask;
            j++;
        }
        const uint64_t m8 = 0x0101010101010101ull * mask;
        for (; c + 8 <= cols; c += 8, j += 8) {             /* whole words, little endian */
            const uint64_t w = mix64(key + ((j >> 3) + 1) * gamma) & m8;
            memcpy(out + c, &w, 8);
        }
        for (; c < cols; c++, j++)                          /* tail */
            out[c] = (uint8_t)(mix64(key + ((j >> 3) + 1) * gamma) >> (8 * (j & 7))) & mask;
    }
}

struct job {
    uint8_t *dst;
    size_t r0, r1, cols;
    uint64_t key, base, row_stride;
    uint8_t mask;
};

static void *run(void *p)
{
    struct job *J = (struct job *)p;
    fill_rows(J->dst, J->r0, J->r1, J->cols, J->key, J->base, J->row_stride, J->mask);
    return NULL;
}

/* rows x cols bytes; a 1-D range is rows = 1 (split into pieces for threads) */
int si_fill_2d(uint8_t *dst, size_t rows, size_t cols, uint64_t seed, uint64_t stream, uint64_t base,
               uint64_t row_stride, uint8_t mask, int threads)
{
    const uint64_t key = seed ^ (stream * 0xD1B54A32D192ED03ull);
    if (rows == 0 || cols == 0) return 0;
    if (threads < 1) threads = 1;
    if (threads > 64) threads = 64;
    if (rows == 1 && cols >= (size_t)threads * 4096) {     /* split one long row into 8-aligned pieces */
        pthread_t th[64];
        struct job J[64];
        const size_t piece = ((cols / threads) + 7) & ~(size_t)7;
        int n = 0;
        for (size_t c0 = 0; c0 < cols && n < 64; c0 += piece, n++) {
            const size_t len = cols - c0 < piece ? cols - c0 : piece;
            J[n] = (struct job){dst + c0, 0, 1, len, key, base + c0, 0, mask};
            if (pthread_create(&th[n], NULL, run, &J[n]) != 0) { run(&J[n]); th[n] = 0; }
        }
        for (int t = 0; t < n; t++)
            if (th[t]) pthread_join(th[t], NULL);
        return 0;
    }
    if (rows < (size_t)threads) threads = (int)rows;
    pthread_t th[64];
    struct job J[64];
    for (int t = 0; t < threads; t++) {
        J[t] = (struct job){dst, rows * t / threads, rows * (t + 1) / threads, cols, key, base, row_stride, mask};
        if (pthread_create(&th[t], NULL, run, &J[t]) != 0) { run(&J[t]); th[t] = 0; }
    }
    for (int t = 0; t < threads; t++)
        if (th[t]) pthread_join(th[t], NULL);
    return 0;
}
