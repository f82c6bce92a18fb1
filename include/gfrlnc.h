/*
 * gfrlnc.h -- C ABI of the B200-native (sm_100a) GF(2^w) region multiply-add
 * and RLNC encoder: the hot path of arXiv 1909.02871 (Guenther, Appel, Carle,
 * "Galois Field Arithmetics for Linear Network Coding using AVX 512
 * Instruction Set Extensions").  Citations "PAPER.md:L" are lines of the
 * paper's LaTeX source; readings "Xn" are listed in DESIGN.md.
 *
 * Conventions shared by every entry point
 *   field   one of 2, 4, 16, 256: F_q with q = 2^w, w in {1,2,4,8}
 *           (Sec. II).  Reduction polynomials x^2+x+1,
 *           x^4+x+1, x^8+x^4+x^3+x+1 (0x11B) (reading X1).
 *   bytes   regions are byte arrays; a byte packs 8/w words, word j at bits
 *           [j*w, (j+1)*w) (reading X4).  Sizes (`bytes`, `M`)
 *           count BYTES, not words: paper M = bytes * 8 / w (reading X10).
 *   memory  every buffer pointer is a CUDA device pointer valid on the current
 *           device, unless the name ends in _host.  The caller owns all
 *           buffers; the library keeps no pointer after a call returns.  Any
 *           alignment and any length are accepted (reading X6).
 *   streams work is enqueued asynchronously on the calling thread's stream
 *           (gf_set_stream; default: the legacy default stream).  Calls that
 *           write disjoint destinations may run concurrently.
 *   errors  every entry point returns a status code (GF_OK == 0); nothing
 *           throws across the ABI.  A size of zero returns GF_OK and launches
 *           nothing.  GF_ECUDA reports a launch / runtime failure
 *           (cudaGetLastError after the launch).
 *   hot path  no allocation, no host synchronisation, no host<->device copy,
 *           no lock and no kernel-attribute call inside gf_maddrc / gf_mulrc /
 *           gf_encode_batch (and gf_invert_batch / gf_decode_batch /
 *           gf_verify_batch): gf_init prepares everything once per (device,
 *           field), so these calls may be captured into a CUDA graph.  (The
 *           TMEM engine encodes a TMA tensor map of A on the host per launch:
 *           host-only work, no driver round trip.)
 */
#ifndef GFRLNC_H
#define GFRLNC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    GF_OK = 0,
    GF_EFIELD = -1,    /* field not in {2, 4, 16, 256}                          */
    GF_ECOEFF = -2,    /* coeff >= q in gf_maddrc / gf_mulrc                    */
    GF_EARG = -3,      /* NULL pointer with nonzero size, N < 1, K < 1, overflow */
    GF_EOVERLAP = -4,  /* partial overlap of dst/src, or B overlapping A or C   */
    GF_ENOINIT = -5,   /* gf_init(field) not called on the current device       */
    GF_ECUDA = -6      /* CUDA launch / runtime failure                          */
};

/* Build the per-coefficient split multiplication tables of F_q on the host
 * and upload them to the CURRENT device (Alg. 1 tables tl/th,
 * re-cut for the GPU into three byte-permute tables), and
 * prepare the field's kernels on that device (dynamic shared-memory opt-ins,
 * the product-row kernel's shared-window probe, the TMEM engine's tensor-map
 * encoder from the driver).  Allocates and synchronises
 * (not a hot-path call).  Idempotent and thread-safe; call once per (device,
 * field) before any other call for that field.  Returns GF_OK, GF_EFIELD or
 * GF_ECUDA. */
int gf_init(int field);

/* Region multiply-add  dst[j] := dst[j] + coeff * src[j]  for j < bytes:
 * the paper's "multiply and add (madd)" b := b + c_i a_i (PAPER.md:91-92,
 * Sec. II; Alg. 1, Alg. 2).
 *   coeff == 0 launches nothing, coeff == 1 runs the XOR kernel
 *   (PAPER.md:205-211 trivial cases).  dst == src (exact aliasing) is allowed
 *   and gives (1 + coeff) * src; any partial overlap returns GF_EOVERLAP.
 * Returns GF_OK, GF_EFIELD, GF_ECOEFF, GF_EARG, GF_EOVERLAP, GF_ENOINIT,
 * GF_ECUDA. */
int gf_maddrc(int field, uint8_t *dst, const uint8_t *src, uint8_t coeff, size_t bytes);

/* Region scaling  dst[j] := coeff * dst[j]  (SPEC mul_region; reading X19).
 * coeff == 1 launches nothing; coeff == 0 zeroes the region. */
int gf_mulrc(int field, uint8_t *dst, uint8_t coeff, size_t bytes);

/* Batched RLNC encode, Eq. 2 over `batch` generations:
 *     B[g][k][m] = sum_{i<N} C[g][i][k] * A[g][i][m]
 * for g < batch, k < K, m < M (byte columns).  Layouts (row-major, packed):
 *     A[batch][N][M]  source packets a_i of generation g (Eq. 1)
 *     C[batch][N][K]  one coding vector c per coded packet, one byte per
 *                     coefficient (readings X9, X11)
 *     B[batch][K][M]  coded packets b, OVERWRITTEN (zero accumulator, X8).
 * Entries of C are not validated on the hot path: a byte >= q is taken
 * modulo q by masking with q-1 (the Python layer offers a checked mode).
 * B must not overlap A or C (GF_EOVERLAP).  Returns GF_OK, GF_EFIELD,
 * GF_EARG, GF_EOVERLAP, GF_ENOINIT, GF_ECUDA. */
int gf_encode_batch(int field, const uint8_t *A, const uint8_t *C, uint8_t *B,
                    int N, int K, size_t M, size_t batch);

/* Same computation with HOST buffers (A_host, C_host read, B_host written):
 * copies in, encodes and copies out in chunks of generations, overlapping
 * host->device copies, kernels and device->host copies on three internal
 * streams.  dev_ws / ws_bytes is a caller-owned device workspace; it must
 * hold at least three chunks of one generation (3 * (N*M + N*K + K*M) + 144
 * bytes); larger workspaces give larger chunks.
 * Pinned host memory is strongly recommended.  BLOCKING: returns after B_host
 * is complete (the caller's stream is not used).  Returns the codes of
 * gf_encode_batch, or GF_EARG when the workspace is too small. */
int gf_encode_batch_host(int field, const uint8_t *A_host, const uint8_t *C_host,
                         uint8_t *B_host, int N, int K, size_t M, size_t batch,
                         void *dev_ws, size_t ws_bytes);

/* Batched inversion of the coefficient matrices (decoder support, SURVEY.md
 * 8(f) NEXT-3; SPEC decode): for g < batch, D[g] = C[g]^{-1} over F_q, i.e.
 * sum_k C[g][i][k] D[g][k][j] = [i == j], by Gauss-Jordan elimination with
 * first-nonzero pivoting.  C, D: [batch][N][N] device bytes (entries masked
 * with q-1), 1 <= N <= 256.  rank (device int[batch], may be NULL) receives
 * the rank of each C[g]; where it is < N, D[g] is unspecified.  Returns
 * GF_OK, GF_EFIELD, GF_ENOINIT, GF_EARG, GF_EOVERLAP, GF_ECUDA. */
int gf_invert_batch(int field, const uint8_t *C, uint8_t *D, int *rank, int N, size_t batch);

/* Batched RLNC decode: recover the N source packets of every generation from
 * N coded packets, closing Eq. 2.  B[batch][N][M] holds the
 * coded packets, C[batch][N][N] their coding vectors in the layout
 * gf_encode_batch uses (C[g][i][k] = coefficient of source i in coded packet
 * k), A[batch][N][M] receives the sources: A = encode(B, C^{-1}).  dev_ws is a
 * device workspace of at least batch * N * N bytes (the inverses).  rank as in
 * gf_invert_batch; rows of A[g] are unspecified where rank[g] < N.  Returns
 * the codes of gf_encode_batch, or GF_EARG for a short workspace. */
int gf_decode_batch(int field, const uint8_t *B, const uint8_t *C, uint8_t *A, int *rank, int N, size_t M,
                    size_t batch, void *dev_ws, size_t ws_bytes);

/* On-device Freivalds check of an encode result (SURVEY.md 8(c) step 7,
 * 8(f) NEXT-4): for every generation and each of t projection vectors
 * r_j = R[g][:, j] (R: [batch][K][t] device bytes < q, t <= 32),
 *     y1 = sum_i (C r_j)_i a_i   and   y2 = sum_k (r_j)_k b_k
 * are formed with the encode kernels (K' = t, so the column kernel) and
 * compared; mismatch[g] (device unsigned long long[batch]) receives the number
 * of differing bytes.  B == A C implies zero; a wrong byte survives one
 * projection with probability <= 1/q.  dev_ws must hold
 * batch*N*t + 2*batch*t*M bytes (+48 for alignment).  Returns the codes of
 * gf_encode_batch, or GF_EARG (t out of range, short workspace). */
int gf_verify_batch(int field, const uint8_t *A, const uint8_t *C, const uint8_t *B, const uint8_t *R, int t,
                    int N, int K, size_t M, size_t batch, unsigned long long *mismatch, void *dev_ws,
                    size_t ws_bytes);

/* Encode with a Freivalds check:
 * B = A C exactly as gf_encode_batch, and for every generation g
 *     mismatch[g] = sum over j < t and blocks b of 64 coded packets of
 *                   #{ m : y1_jb[m] != y2_jb[m] },
 *     y2_jb = sum_{k in b} r_jk b_k,   y1_jb = sum_i u_jbi a_i,
 *     u_jbi = sum_{k in b} r_jk C[g][i][k]          (Eq. 2 projected on r_j)
 * with BINARY projection vectors r_jk = R[g][k][j] & 1 (R: [batch][K][t]
 * device bytes, t in {1, 2}).  B == A C gives 0; a wrong byte of B escapes one
 * projection with probability <= 1/2 for uniform random r.  The GF(2) split
 * engine (K <= 64: C5 GF(2)) and the lane-k kernel (K <= 64: C5 GF(4)) check
 * inside the encode -- the coded words while they are still on chip, the
 * source words they already hold (both are HBM-heavy, so no second pass over
 * A and B); every other kernel (the product-row kernels of C3 / C4 among them)
 * runs the encode and then one streaming pass over A and B in the same call,
 * on the same stream.  dev_ws: 16-byte
 * aligned device workspace of at least
 *     round16(batch * ceil(K/64) * 2 * N) + batch * 2 * ceil(K/32) * 4 bytes.
 * Returns the codes of gf_encode_batch, or GF_EARG (t, R, mismatch, workspace,
 * batch > 2^31 - 1 or K > 196608). */
int gf_encode_verify_batch(int field, const uint8_t *A, const uint8_t *C, uint8_t *B, const uint8_t *R, int t,
                           int N, int K, size_t M, size_t batch, unsigned long long *mismatch, void *dev_ws,
                           size_t ws_bytes);

/* Set the calling thread's stream (a cudaStream_t; NULL = legacy default). */
int gf_set_stream(void *cuda_stream);

/* Static description of a status code; never NULL. */
const char *gf_strerror(int status);

/* ---- harness-only exports (not part of the paper's method) -------------- */

/* Counter-based generator shared with seeded_inputs:
 *   byte(seed, stream, j) = byte (j & 7) of
 *       mix64((seed ^ stream * 0xD1B54A32D192ED03) + ((j >> 3) + 1) * 0x9E3779B97F4A7C15)
 * gf_fill_random:   dst[j] = byte(seed, stream, offset + j) & mask, j < bytes
 * gf_fill_random2d: dst[r*cols + c] = byte(seed, stream, base + r*row_stride + c) & mask
 * mask = 0xFF for payload bytes, q-1 for coefficients uniform over F_q. */
int gf_fill_random(uint8_t *dst, size_t bytes, uint64_t seed, uint64_t stream,
                   uint64_t offset, uint8_t mask);
int gf_fill_random2d(uint8_t *dst, size_t rows, size_t cols, uint64_t seed, uint64_t stream,
                     uint64_t base, uint64_t row_stride, uint8_t mask);

/* Host-only (no GPU needed): copy out the per-coefficient tables gf_init
 * uploads, so CPU tests can emulate the kernels' arithmetic.  Writes
 * q * 16 uint32 words: for coefficient c, words [16c .. 16c+15] =
 *   { T0[0..3], T0[4..7], T1[0..3], T1[4..7], T2[0..3], M0, M1, 0,
 *     pow[c][0], ..., pow[c][7] }
 * with Tg[v] = c * (v << 3g) (packed product, one byte per entry, little
 * endian; byte-permute split tables, GPU form of Alg. 1's tl/th), M0/M1 the
 * all-ones masks of coefficient bits 0/1 (GF(2)/GF(4) bit planes), and
 * pow[c][j] = c * x^j for j < w, else 0 (Alg. 2's imul constants,
 * PAPER.md:245,266).  Returns GF_OK, GF_EFIELD or GF_EARG (cap too small). */
int gf_host_tables(int field, uint32_t *out, size_t cap_words);

/* Host-only introspection (harness / roofline accounting): which encode kernel
 * gf_encode_batch launches for these arguments, given the byte offsets of A
 * and B modulo 16.  Returns 0 = column kernel on 32-bit words, 1 = column
 * kernel on bytes (unaligned or M % 4 != 0), 2 / 3 = lane-k kernel with 32 /
 * 64 (128 when K > 64) coded packets per CTA (GF(4), K >= 24, and GF(2) where
 * the split engine does not apply), 6 / 9 / 10 = product-row kernel with 64 /
 * 32 / 16 coded packets per CTA (GF(16)/GF(256), K > 8: C3, C4; GF(4) with
 * 9 <= K < 24 on well-tiled packets), 8 = streaming kernel (K <= 4: C1 and
 * the paper's N = 16, K = 1 shape; its chunk layout -- 16-byte chunks one,
 * two or four per thread, or 4-byte words one or 4 / 8 / 12 strided per
 * thread -- follows from M, the alignment and the job size), 11 = GF(2) split
 * engine (GF(2), K >= 24, N <= 32, M % 16 == 0, 16-byte aligned A and B: C5),
 * 12 = GF(16) product-row kernel with nibble-indexed tables (K > 32: C3 GF(16)),
 * 13 = GF(256) product-row kernel with 32 coded packets per CTA on 768-word
 * tiles (K > 32, packets of >= 6144 words tiled >= 90%: C4)
 * 14 = TMEM lookup-table engine (GF(2) with K >= 9, GF(4) with K >= 5, GF(16) with
 * K >= 5 -- N <= 32 when K > 32, not 13 <= K <= 16 on packets >= 8 KiB;
 * M >= 256, M % 16 == 0, 16-byte aligned A and B: C5)
 * (DESIGN.md section 6), or GF_EFIELD / GF_EARG. */
int gf_encode_path(int field, int N, int K, size_t M, size_t a_align, size_t b_align);

/* Harness-only (forced-path tests and experiments): force the encode kernel of
 * the calling thread's gf_encode_batch calls.  Thread-local; nothing is read
 * from the environment.  Shapes a forced kernel cannot take fall back to the
 * lane-k kernel (GF_PATH_GF2: to the automatic choice).  Returns GF_OK or
 * GF_EARG. */
enum {
    GF_PATH_AUTO = 0,
    GF_PATH_COLUMN = 1,
    GF_PATH_LANEK = 2,
    GF_PATH_PROW = 4,
    GF_PATH_STREAM = 6,              /* streaming kernel, automatic layout      */
    GF_PATH_GF2 = 7,                 /* GF(2) split engine                      */
    GF_PATH_STREAM_STRIDED4 = 8,     /* streaming, strided 4-word blocks at any job size */
    GF_PATH_STREAM_STRIDED8 = 9,     /* ... 8-word blocks                       */
    GF_PATH_STREAM_STRIDED12 = 10,   /* ... 12-word blocks                      */
    GF_PATH_STREAM_WIDE2 = 11,       /* streaming, two 16-byte chunks per thread at any packet size */
    GF_PATH_STREAM_WIDE4 = 12,       /* streaming, four 16-byte chunks per thread                   */
    GF_PATH_TMEM = 13                /* TMEM lookup-table engine (any field; M % 16 == 0, 16-byte aligned) */
};
int gf_set_encode_path(int path);

/* Harness-only (tests of the check): make the calling thread's next
 * gf_encode_verify_batch calls corrupt one byte (XOR 0x5A) of coded packet k,
 * 32-bit word `word`, of generation g -- in the kernel before the store and
 * the projection (GF(2) split engine, lane-k) or in B after the encode (other
 * paths).
 * enable = 0 turns it off.  Returns GF_OK or GF_EARG. */
int gf_set_verify_fault(int enable, size_t g, int k, size_t word);

/* Library version (major * 10000 + minor * 100 + patch). */
int gf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GFRLNC_H */
