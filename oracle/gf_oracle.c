/*
 * gf_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 1909.02871 (Guenther, Appel, Carle: "Galois Field Arithmetics for
 * Linear Network Coding using AVX 512 Instruction Set Extensions").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1909_02871_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Compiled with -O2 -fno-tree-vectorize: scalar code, no SIMD, no blocking.
 *
 * What it computes (citations are PAPER.md line numbers + section/equation):
 *   - F_q elements, q in {2,4,16,256}, are polynomials over GF(2), bit k being
 *     the coefficient of x^k (Sec. II; reading X3 in DESIGN.md).
 *   - addition is XOR, multiplication is the polynomial product reduced modulo
 *     a field-specific polynomial (Sec. II).  The paper never names
 *     the polynomials; we take x^2+x+1, x^4+x+1, x^8+x^4+x^3+x+1 (reading X1).
 *   - a byte packs 8/w words of w bits, word j at bits [j*w,(j+1)*w)
 *     (reading X4).
 *   - madd: b := b + c*a over a region (Sec. II; Alg. 1/2
 *     PAPER.md:197-294).  mulrc: b := c*b (reading X19, SPEC mul_region).
 *   - encode: b = A c = sum_i c_i a_i (Eq. 2), batched to
 *     B[g][k][m] = sum_i C[g][i][k] * A[g][i][m] over many generations
 *     (readings X8, X9, X10 in DESIGN.md).
 *   - Freivalds projection check, Gauss-Jordan rank/solve (test tools, not the
 *     paper's method).
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---- field description (Sec. II; polynomials = reading X1) */

/* returns w = log2(q), or -1 for an unsupported q */
int gfo_width(int q)
{
    switch (q) {
    case 2: return 1;
    case 4: return 2;
    case 16: return 4;
    case 256: return 8;
    default: return -1;
    }
}

/* reduction polynomial including the leading x^w term (reading X1).
 * GF(2): x+1 -- any degree-1 polynomial, never used because a product of two
 * 1-bit values has degree 0. */
unsigned gfo_poly(int q)
{
    switch (q) {
    case 2: return 0x3u;    /* x + 1 */
    case 4: return 0x7u;    /* x^2 + x + 1 */
    case 16: return 0x13u;  /* x^4 + x + 1 */
    case 256: return 0x11Bu;/* x^8 + x^4 + x^3 + x + 1 */
    default: return 0u;
    }
}

/* ---- element multiplication, formulation 1: schoolbook carry-less product,
 * then reduction from the top degree down ("multiplication is a
 * modulo operation given a reduction polynomial").                          */
unsigned gfo_poly_mul(int q, unsigned a, unsigned b)
{
    int w = gfo_width(q);
    unsigned P = gfo_poly(q);
    unsigned r = 0;
    int k, d;
    if (w < 0) return 0;
    for (k = 0; k < w; k++)
        if ((b >> k) & 1u)
            r ^= a << k;                 /* add a * x^k */
    for (d = 2 * w - 2; d >= w; d--)
        if ((r >> d) & 1u)
            r ^= P << (d - w);           /* subtract P * x^(d-w) */
    return r;
}

/* ---- element multiplication, formulation 2 (independent): scan the bits of
 * b from x^0 upwards, keeping t = a * x^k reduced at every step ("xtime").  */
unsigned gfo_poly_mul_xtime(int q, unsigned a, unsigned b)
{
    int w = gfo_width(q);
    unsigned P = gfo_poly(q);
    unsigned r = 0, t = a;
    int k;
    if (w < 0) return 0;
    for (k = 0; k < w; k++) {
        if ((b >> k) & 1u)
            r ^= t;
        t <<= 1;                          /* t := t * x */
        if ((t >> w) & 1u)
            t ^= P;                       /* reduce the x^w term */
    }
    return r;
}

/* multiplicative inverse by exhaustive search (SPEC gf_inv); 0 for a == 0 */
unsigned gfo_inv(int q, unsigned a)
{
    unsigned x;
    if (a == 0) return 0;
    for (x = 1; x < (unsigned)q; x++)
        if (gfo_poly_mul(q, a, x) == 1u)
            return x;
    return 0;
}

/* ---- packed byte multiply: every w-bit word of v multiplied by c
 * (PAPER.md:57-61 words in a byte; reading X4 for the slot order).          */
unsigned gfo_mulbyte(int q, unsigned c, unsigned v)
{
    int w = gfo_width(q);
    unsigned mask = (unsigned)q - 1u, out = 0;
    int j;
    if (w < 0) return 0;
    for (j = 0; j < 8 / w; j++) {
        unsigned word = (v >> (j * w)) & mask;
        out |= gfo_poly_mul(q, c, word) << (j * w);
    }
    return out & 0xFFu;
}

/* MB[c*256 + v] = mulbyte(c, v) for c < q, v < 256.  Returns 0 on success,
 * -1 if any entry disagrees with formulation 2 (self-check). */
int gfo_build_mb(int q, uint8_t *MB)
{
    int w = gfo_width(q);
    unsigned c, v;
    if (w < 0) return -1;
    for (c = 0; c < (unsigned)q; c++)
        for (v = 0; v < 256u; v++) {
            unsigned x = gfo_mulbyte(q, c, v), y = 0;
            int j;
            for (j = 0; j < 8 / w; j++)
                y |= gfo_poly_mul_xtime(q, c, (v >> (j * w)) & ((unsigned)q - 1u)) << (j * w);
            if (x != y) return -1;
            MB[c * 256u + v] = (uint8_t)x;
        }
    return 0;
}

/* per-q cached tables (built on first use; deterministic) */
static uint8_t g_mb[4][256 * 256];
static int g_mb_ready[4];
static pthread_mutex_t g_mb_lock = PTHREAD_MUTEX_INITIALIZER;

static int qidx(int q)
{
    switch (q) { case 2: return 0; case 4: return 1; case 16: return 2; case 256: return 3; }
    return -1;
}

static const uint8_t *mb_table(int q)
{
    int i = qidx(q);
    if (i < 0) return NULL;
    pthread_mutex_lock(&g_mb_lock);
    if (!g_mb_ready[i]) {
        if (gfo_build_mb(q, g_mb[i]) != 0) { pthread_mutex_unlock(&g_mb_lock); return NULL; }
        g_mb_ready[i] = 1;
    }
    pthread_mutex_unlock(&g_mb_lock);
    return g_mb[i];
}

/* ---- region operations (PAPER.md:91-92 madd; Alg. 1) ---- */

/* dst[j] ^= c * src[j]  (b := b + c a).  Returns 0, or -1 on bad q / c. */
int gfo_maddrc(int q, uint8_t *dst, const uint8_t *src, unsigned c, size_t n)
{
    const uint8_t *MB = mb_table(q);
    size_t j;
    if (!MB || c >= (unsigned)q) return -1;
    for (j = 0; j < n; j++)
        dst[j] ^= MB[c * 256u + src[j]];
    return 0;
}

/* dst[j] = c * dst[j] */
int gfo_mulrc(int q, uint8_t *dst, unsigned c, size_t n)
{
    const uint8_t *MB = mb_table(q);
    size_t j;
    if (!MB || c >= (unsigned)q) return -1;
    for (j = 0; j < n; j++)
        dst[j] = MB[c * 256u + dst[j]];
    return 0;
}

/* ---- encode (Eq. 2), one generation, byte columns
 * [m0, m1) of each packet:
 *   out[k*(m1-m0) + (m-m0)] = XOR_i mulbyte(C[i*K + k], A[i*lda + m])
 * A points at packet 0 of the generation, lda = bytes between packets.      */
int gfo_encode_gen_cols(int q, const uint8_t *A, size_t lda, const uint8_t *C,
                        uint8_t *out, int N, int K, size_t m0, size_t m1)
{
    const uint8_t *MB = mb_table(q);
    size_t m, w = m1 - m0;
    int i, k;
    if (!MB || N < 1 || K < 1 || m1 < m0) return -1;
    for (k = 0; k < K; k++)
        for (m = m0; m < m1; m++) {
            unsigned acc = 0;
            for (i = 0; i < N; i++)
                acc ^= MB[(unsigned)C[(size_t)i * K + k] * 256u + A[(size_t)i * lda + m]];
            out[(size_t)k * w + (m - m0)] = (uint8_t)acc;
        }
    return 0;
}

/* B[g][k][m] = XOR_i C[g][i][k] * A[g][i][m] for all g < batch (B overwritten,
 * reading X8).  Layouts: A[batch][N][M], C[batch][N][K], B[batch][K][M]. */
int gfo_encode_batch(int q, const uint8_t *A, const uint8_t *C, uint8_t *B,
                     int N, int K, size_t M, size_t batch)
{
    size_t g;
    for (g = 0; g < batch; g++) {
        int rc = gfo_encode_gen_cols(q, A + g * (size_t)N * M, M, C + g * (size_t)N * K,
                                     B + g * (size_t)K * M, N, K, 0, M);
        if (rc) return rc;
    }
    return 0;
}

/* same, generations split over nthreads host threads (harness: timing only) */
struct enc_job {
    int q, N, K; size_t M, g0, g1;
    const uint8_t *A, *C; uint8_t *B; int rc;
};

static void *enc_worker(void *p)
{
    struct enc_job *j = (struct enc_job *)p;
    j->rc = gfo_encode_batch(j->q, j->A + j->g0 * (size_t)j->N * j->M,
                             j->C + j->g0 * (size_t)j->N * j->K,
                             j->B + j->g0 * (size_t)j->K * j->M,
                             j->N, j->K, j->M, j->g1 - j->g0);
    return NULL;
}

int gfo_encode_batch_mt(int q, const uint8_t *A, const uint8_t *C, uint8_t *B,
                        int N, int K, size_t M, size_t batch, int nthreads)
{
    struct enc_job jobs[256];
    pthread_t th[256];
    int t, rc = 0;
    if (!mb_table(q)) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((size_t)nthreads > batch) nthreads = batch ? (int)batch : 1;
    for (t = 0; t < nthreads; t++) {
        jobs[t].q = q; jobs[t].N = N; jobs[t].K = K; jobs[t].M = M;
        jobs[t].g0 = batch * (size_t)t / (size_t)nthreads;
        jobs[t].g1 = batch * (size_t)(t + 1) / (size_t)nthreads;
        jobs[t].A = A; jobs[t].C = C; jobs[t].B = B; jobs[t].rc = 0;
        pthread_create(&th[t], NULL, enc_worker, &jobs[t]);
    }
    for (t = 0; t < nthreads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc) rc = jobs[t].rc;
    }
    return rc;
}

/* ---- Freivalds projection check --------------
 * For one generation and one random r in F_q^K (given as K bytes < q):
 *   u = C r (N values), y1 = sum_i u_i a_i, y2 = sum_k r_k b_k  (M bytes each)
 * and counts byte positions where y1 != y2.  B == A C implies y1 == y2; a
 * wrong word survives one projection with probability <= 1/q.               */
long gfo_freivalds_gen(int q, const uint8_t *A, const uint8_t *C, const uint8_t *B,
                       int N, int K, size_t M, const uint8_t *r, uint8_t *scratch2M)
{
    const uint8_t *MB = mb_table(q);
    uint8_t *y1 = scratch2M, *y2 = scratch2M + M;
    long bad = 0;
    size_t m;
    int i, k;
    if (!MB) return -1;
    memset(y1, 0, M);
    memset(y2, 0, M);
    for (i = 0; i < N; i++) {
        unsigned u = 0;                      /* u_i = sum_k C[i][k] r_k (packed byte product) */
        for (k = 0; k < K; k++)
            u ^= MB[(unsigned)C[(size_t)i * K + k] * 256u + r[k]];
        /* r_k and C entries are single field elements (< q), so u < q */
        gfo_maddrc(q, y1, A + (size_t)i * M, u, M);
    }
    for (k = 0; k < K; k++)
        gfo_maddrc(q, y2, B + (size_t)k * M, r[k], M);
    for (m = 0; m < M; m++)
        bad += (y1[m] != y2[m]);
    return bad;
}

/* ---- Gauss-Jordan over F_q (test tool: SPEC rank/decode, NEXT-3) -------
 * Mx is rows x cols bytes, row-major.  The first ecols columns hold single
 * field elements (< q) and are the pivot columns; the remaining columns may
 * hold packed payload bytes.  Every row operation multiplies whole bytes with
 * mulbyte, which equals the element product on the element columns (a value
 * < q occupies word slot 0 only).  Returns the rank of the element block and
 * leaves it in reduced row echelon form.                                     */
int gfo_rref(int q, uint8_t *Mx, int rows, int cols, int ecols)
{
    const uint8_t *MB = mb_table(q);
    int r = 0, c, i, j;
    if (!MB || ecols > cols) return -1;
    for (c = 0; c < ecols && r < rows; c++) {
        int piv = -1;
        unsigned inv;
        for (i = r; i < rows; i++)
            if (Mx[(size_t)i * cols + c]) { piv = i; break; }
        if (piv < 0) continue;
        if (piv != r)
            for (j = 0; j < cols; j++) {
                uint8_t t = Mx[(size_t)r * cols + j];
                Mx[(size_t)r * cols + j] = Mx[(size_t)piv * cols + j];
                Mx[(size_t)piv * cols + j] = t;
            }
        inv = gfo_inv(q, Mx[(size_t)r * cols + c]);
        for (j = 0; j < cols; j++)
            Mx[(size_t)r * cols + j] = MB[inv * 256u + Mx[(size_t)r * cols + j]];
        for (i = 0; i < rows; i++) {
            unsigned f = Mx[(size_t)i * cols + c];
            if (i == r || f == 0) continue;
            for (j = 0; j < cols; j++)
                Mx[(size_t)i * cols + j] ^= MB[f * 256u + Mx[(size_t)r * cols + j]];
        }
        r++;
    }
    return r;
}
