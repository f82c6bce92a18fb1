// encode_gf2.cuh -- batched RLNC encode over GF(2) with the source words of a
// 512-byte column span held in registers and the multiply-add of every
// (source i, coded packet k) split between the two integer pipes.
//
//   B[g][k][m] = XOR_{i < N} C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Over GF(2) a coefficient is one bit, so c * a is either a or 0 for a whole
// 32-bit word of 32 field elements ("GF(2): XOR").  Two
// data-independent ways to apply it, on two different pipes:
//   * masked XOR on the ALU pipe: acc ^= a & m with m = 0 or ~0 (one LOP3 per
//     term -- the paper's bit-plane masking, Alg. 2's `and` step);
//   * the paper's imul (Alg. 2) on the FMA pipe: a * c with
//     c = 0 or 1 is one IMAD; two such products are folded into the
//     accumulator by one 3-input LOP3 (acc ^ p0 ^ p1).
// Sources i with i % 3 == 2 take the masked form, the others the imul form in
// pairs, so per (word, coded packet) the 32 terms cost 21 ALU + 22 FMA
// instructions: both pipes ~2/3 busy per term and 1.34 issue slots per term
// (all-masked would be 1 issue slot but 1 ALU op per term, ALU-bound at 71% of
// the HBM roofline; tools/exp_c5_branch.cu has both and the branch variants).
//
// Layout: a block (4 warps) owns one generation; its coefficient words
// cw[k][i] (c or mask, per the form of source i) are built once into shared
// memory and read back per coded packet with broadcast LDS.128.  Lane l of a
// warp owns words w0 + 4l .. w0 + 4l + 3 of every packet of a 128-word span
// (16-byte loads / stores, 512 contiguous bytes per warp per packet); all NS
// source words of the span stay in registers (4 NS registers) while the warp
// walks k = 0 .. K-1 and stores each coded packet's span once.  HBM traffic is
// the algorithmic N*M + K*M (+ N*K) per generation.
//
// Requirements (checked by the router): 1 <= N <= NS, M % 16 == 0, A and B
// 16-byte aligned.  Sources i >= N get zero coefficients.
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kG2Threads = 128;            // 4 warps, one generation per block
constexpr int kG2SpanWords = 128;          // 32 lanes x 4 words

struct Gf2Params {
    const uint8_t *A;      // [batch][N][M]
    const uint8_t *C;      // [batch][N][K]
    uint8_t *B;            // [batch][K][M]
    uint32_t Mw;           // 32-bit words per packet (M / 4, M % 16 == 0)
    uint32_t spans;        // 128-word spans per packet
    int spw;               // spans per warp
    int N, K;
    // fused Freivalds check (T > 0 instantiations; gf_encode_verify_batch)
    const uint8_t *U;      // [batch][1][2][N]: u_j = C r_j (bit 0), r_j binary
    const uint32_t *RB;    // [batch][2][kw]: bit k of word k / 32 = r_jk
    int kw;                // 32-bit words per RB row: ceil(K / 32)
    int t;                 // projections in use (1 or 2)
    unsigned long long *mismatch;   // [batch] += differing bytes
    uint64_t fault;        // harness fault injection: bit 63 on, g << 32 | k << 20 | word
};


__device__ __forceinline__ uint4 g2_ld(const uint8_t *p)
{
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// predicated streaming store (no branch, so no reconvergence barrier in the k
// loop; .cs: B is written once and not re-read: +0.4%, profiles/r02_gf2_cs.txt)
__device__ __forceinline__ void g2_st(uint8_t *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t on)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %5, 0;\n\t@q st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};\n\t}"
                 :: "l"(p), "r"(a), "r"(b), "r"(c), "r"(d), "r"(on) : "memory");
}

// FULL: N == NS (no clamped source addresses).  Grid: x = block within the
// generation (4 warps x spw spans each), y = generation (offset g_base, so that
// more than 65535 generations take several launches).
//
// T = 2: the fused Freivalds check of gf_encode_verify_batch (SURVEY 8(c) step
// 7, 8(f) NEXT-4) on binary projection vectors r_j (j < t): while a coded
// packet's words are still in registers, y2_j ^= b_k & -(r_jk) (one LOP3 per
// projection and word); once per span, y1_j = XOR_i a_i & -(u_ji) with
// u_j = C r_j from the source words already in registers; then the bytes
// where y1_j != y2_j are counted into mismatch[g].  B == A C gives zero; a
// wrong byte escapes one binary projection with probability <= 1/2.
// FT: the harness fault injection (gf_set_verify_fault) -- a separate
// instantiation, so the production check carries no per-row test code.
template <int NS, bool FULL, int T = 0, bool FT = false>
__global__ void __launch_bounds__(kG2Threads, T > 0 ? 3 : 1) encode_gf2_kernel(Gf2Params p, uint32_t g_base)
{
    extern __shared__ __align__(16) uint32_t cw[];              // [K][NS] (+ T: mr [K][T], mu [T][NS])
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t g = (size_t)g_base + blockIdx.y;
    const int N = FULL ? NS : p.N, K = p.K;
    uint32_t *mr = cw + K * NS, *mu = mr + K * T;
    {
        const uint8_t *Cg = p.C + g * (size_t)N * K;
        for (int t = threadIdx.x; t < K * NS; t += kG2Threads) {
            const int k = t / NS, i = t - k * NS;
            const uint32_t c = (FULL || i < N) ? (__ldg(Cg + (size_t)i * K + k) & 1u) : 0u;
            cw[t] = (i % 3 == 2) ? 0u - c : c;              // mask for the ALU form, 0/1 for imul
        }
        if constexpr (T > 0) {
            for (int e = threadIdx.x; e < K * T; e += kG2Threads) {
                const int k = e / T, j = e - k * T;
                mr[e] = j < p.t ? 0u - ((__ldg(p.RB + (g * 2 + j) * p.kw + (k >> 5)) >> (k & 31)) & 1u) : 0u;
            }
            for (int e = threadIdx.x; e < T * NS; e += kG2Threads) {
                const int j = e / NS, i = e - j * NS;
                mu[e] = (j < p.t && i < N) ? 0u - (__ldg(p.U + (g * 2 + j) * (size_t)N + i) & 1u) : 0u;
            }
        }
    }
    __syncthreads();
    uint32_t bad = 0;
    const uint32_t Mw = p.Mw;
    const uint32_t sp0 = (blockIdx.x * 4 + wid) * (uint32_t)p.spw;
#pragma unroll 1
    for (int s = 0; s < p.spw; s++) {
        const uint32_t sp = sp0 + s;
        if (sp >= p.spans) break;
        const uint32_t w0 = sp * kG2SpanWords + 4 * lane;
        const bool valid = w0 < Mw;
        // sources i >= N re-read source 0 (their coefficients are zero, so any
        // value gives a zero term); lanes past the packet end read word 0 and
        // never store
        const uint32_t *Ag = reinterpret_cast<const uint32_t *>(p.A) + g * (size_t)N * Mw + (valid ? w0 : 0u);
        uint32_t a[NS][4];
#pragma unroll
        for (int i = 0; i < NS; i++) {
            const uint4 v = g2_ld(reinterpret_cast<const uint8_t *>(Ag + (size_t)(FULL || i < N ? i : 0) * Mw));
            a[i][0] = v.x; a[i][1] = v.y; a[i][2] = v.z; a[i][3] = v.w;
        }
        uint32_t *Bg = reinterpret_cast<uint32_t *>(p.B) + g * (size_t)K * Mw + w0;
        // harness fault injection: the coded packet to corrupt if this lane holds the word
        const int fk = (FT && g == ((p.fault >> 32) & 0x7FFFFFFFu) && w0 == ((uint32_t)p.fault & 0xFFFFCu))
                           ? (int)((p.fault >> 20) & 0xFFFu) : -1;
        (void)fk;
        uint32_t y2[T > 0 ? T : 1][4];
#pragma unroll
        for (int j = 0; j < (T > 0 ? T : 1); j++)
#pragma unroll
            for (int w = 0; w < 4; w++) y2[j][w] = 0;
#pragma unroll 1
        for (int k = 0; k < K; k++) {
            uint32_t mk[T > 0 ? T : 1];                // projection masks of row k, loaded with its coefficients
#pragma unroll
            for (int j = 0; j < T; j++) mk[j] = mr[k * T + j];
            (void)mk;
            uint32_t c[NS];
#pragma unroll
            for (int q = 0; q < NS / 4; q++) {
                const uint4 v = reinterpret_cast<const uint4 *>(cw + k * NS)[q];
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
            uint32_t acc[4];
#pragma unroll
            for (int w = 0; w < 4; w++) {
                uint32_t x = 0;
#pragma unroll
                for (int i = 0; i < NS; i += 3) {
                    if (i + 1 < NS) x ^= (a[i][w] * c[i]) ^ (a[i + 1][w] * c[i + 1]);   // 2 IMAD + LOP3
                    else x ^= a[i][w] * c[i];
                    if (i + 2 < NS) x ^= a[i + 2][w] & c[i + 2];                        // LOP3
                }
                acc[w] = x;
            }
            if constexpr (T > 0) {
                if constexpr (FT)
                    if (k == fk) acc[p.fault & 3u] ^= 0x5Au;            // harness: one wrong byte
#pragma unroll
                for (int j = 0; j < T; j++)
#pragma unroll
                    for (int w = 0; w < 4; w++) y2[j][w] ^= acc[w] & mk[j];
            }
            g2_st(reinterpret_cast<uint8_t *>(Bg + (size_t)k * Mw), acc[0], acc[1], acc[2], acc[3],
                  valid ? 1u : 0u);
        }
        if constexpr (T > 0) {                     // y1 from the source words, still in registers
            const uint32_t mus = (uint32_t)__cvta_generic_to_shared(mu);
#pragma unroll
            for (int j = 0; j < T; j++) {
                // two independent XOR chains per word (even / odd source groups),
                // joined at the end: half the dependent-LOP3 depth
                uint32_t x[4] = {y2[j][0], y2[j][1], y2[j][2], y2[j][3]}, xo[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int q = 0; q < NS / 4; q++) {
                    uint4 m;                          // volatile: read here, not hoisted across the k loop
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(m.x), "=r"(m.y), "=r"(m.z), "=r"(m.w) : "r"(mus + (uint32_t)(j * NS + 4 * q) * 4u));
#pragma unroll
                    for (int w = 0; w < 4; w++) {
                        uint32_t &xx = (q & 1) ? xo[w] : x[w];
                        xx ^= a[4 * q][w] & m.x;
                        xx ^= a[4 * q + 1][w] & m.y;
                        xx ^= a[4 * q + 2][w] & m.z;
                        xx ^= a[4 * q + 3][w] & m.w;
                    }
                }
#pragma unroll
                for (int w = 0; w < 4; w++) x[w] ^= xo[w];
                if (valid)
#pragma unroll
                    for (int w = 0; w < 4; w++) bad += nz_bytes(x[w]);
            }
        }
    }
    if constexpr (T > 0) {
        bad = __reduce_add_sync(0xffffffffu, bad);
        if (lane == 0 && bad) atomicAdd(p.mismatch + g, (unsigned long long)bad);
    }
}

__host__ __device__ constexpr size_t gf2_smem_bytes(int K, int NS, int T = 0)
{
    return (size_t)K * NS * 4 + (size_t)T * (K + NS) * 4;
}

}  // namespace gfr
