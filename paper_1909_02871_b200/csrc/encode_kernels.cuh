// encode_kernels.cuh -- batched RLNC encode B = A C over F_q (Eq. 2,
// PAPER.md:84-88), one kernel family per field.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]
//
// Work decomposition:
//   * a warp owns one generation g and a span of 32*W packet words (word =
//     4 bytes; lane l holds words span0 + w*32 + l, w < W, so every warp load
//     and store is a contiguous 128-byte line);
//   * a CTA owns KT coded packets k0 .. k0+KT-1 and either several whole
//     generations (short packets, e.g. M = 1500) or WPB spans of one
//     generation (long packets); the KT index varies fastest over the grid so
//     the CTAs that re-read the same A tile run together and hit L2;
//   * each source word is loaded ONCE per CTA and reused for all KT outputs:
//     the c-independent part of the multiply (PRMT selectors, GF(4) x*a) is
//     computed once per (i, word) and amortised over KT coefficients;
//   * the coefficients of the current chunk of NI source packets are resolved
//     to their lookup tables in shared memory; within a warp they are
//     uniform, so every table read is a broadcast;
//   * accumulators (KT x W words) live in registers for the whole i loop and
//     B is written once (overwrite semantics, reading X8).
//
// Per (i, k, word) the inner loop costs
//   GF(256)/GF(16): 3 PRMT + 2 LOP3  (byte-permute split tables),
//   GF(4):          2 LOP3           (bit planes: c0*a ^ c1*(x a)),
//   GF(2):          1 LOP3           (acc ^= a & mask(c)).
//
// BYTEWISE = true is the generic path for packets whose length is not a
// multiple of 4 or whose rows are not 4-byte aligned: a "word" is then a
// single byte zero-extended into a 32-bit register, which every field kernel
// handles unchanged (a byte in lane 0 is a valid packed word).
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kEncNI = 16;   // source packets per table chunk

struct EncodeParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    const uint32_t *tabs;     // device table of tables, 8 words per coefficient
    size_t M;                 // bytes per packet
    size_t Mw;                // words per packet (M / 4, or M when BYTEWISE)
    size_t batch;
    int N, K;
    int qmask;                // q - 1
    int spans_per_gen;        // ceil(Mw / (32 W))
    int gens_per_cta;         // > 1 only when a CTA holds whole generations
    int ctas_per_gen;         // CTAs along one generation's spans
    int k_tiles;              // ceil(K / KT)
};

template <int F> struct EncTraits;
template <> struct EncTraits<256> { static constexpr int kEntryWords = 5; };
template <> struct EncTraits<16>  { static constexpr int kEntryWords = 5; };
template <> struct EncTraits<4>   { static constexpr int kEntryWords = 2; };
template <> struct EncTraits<2>   { static constexpr int kEntryWords = 1; };

template <int F, int KT>
__host__ __device__ constexpr size_t enc_smem_bytes_per_gen()
{
    return (size_t)kEncNI * KT * EncTraits<F>::kEntryWords * 4u;
}

template <bool BYTEWISE>
__device__ __forceinline__ uint32_t ld_word(const uint8_t *row, size_t word)
{
    if (BYTEWISE) return (uint32_t)__ldg(row + word);
    return __ldg(reinterpret_cast<const uint32_t *>(row) + word);
}

template <bool BYTEWISE>
__device__ __forceinline__ void st_word(uint8_t *row, size_t word, uint32_t v)
{
    if (BYTEWISE) row[word] = (uint8_t)(v & 0xFFu);
    else reinterpret_cast<uint32_t *>(row)[word] = v;
}

template <int F, int W, int KT, bool BYTEWISE>
__global__ void __launch_bounds__(256) encode_kernel(EncodeParams p)
{
    extern __shared__ __align__(16) uint32_t smem[];
    // layout per local generation: [NI][KT] entries; PRMT fields split the
    // entry into a uint4 array (T0, T1) followed by a uint32 array (T2)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;

    const size_t bid = blockIdx.x;
    const int kt = (int)(bid % (size_t)p.k_tiles);
    const size_t rest = bid / (size_t)p.k_tiles;
    const int k0 = kt * KT;
    const int kc = min(KT, p.K - k0);

    size_t g_first;
    int gl, span;
    if (p.gens_per_cta > 1 || p.ctas_per_gen == 1) {
        g_first = rest * (size_t)p.gens_per_cta;
        gl = warp / p.spans_per_gen;
        span = warp % p.spans_per_gen;
    } else {
        g_first = rest / (size_t)p.ctas_per_gen;
        gl = 0;
        span = (int)(rest % (size_t)p.ctas_per_gen) * nwarps + warp;
    }
    const int ngen = (int)min((size_t)p.gens_per_cta, p.batch - g_first);
    const bool active = gl < ngen && span < p.spans_per_gen;
    const size_t g = g_first + (size_t)gl;
    const size_t word0 = (size_t)span * 32u * W + lane;

    uint32_t acc[KT][W];
#pragma unroll
    for (int k = 0; k < KT; k++)
#pragma unroll
        for (int w = 0; w < W; w++) acc[k][w] = 0u;

    const uint8_t *Ag = p.A + (active ? g : 0) * (size_t)p.N * p.M;
    uint32_t cur[W], nxt[W];
#pragma unroll
    for (int w = 0; w < W; w++) {
        const size_t wd = word0 + (size_t)w * 32u;
        cur[w] = (active && wd < p.Mw) ? ld_word<BYTEWISE>(Ag, wd) : 0u;
    }

    uint4 *tab4 = reinterpret_cast<uint4 *>(smem);
    uint32_t *tab1 = smem + (size_t)p.gens_per_cta * kEncNI * KT * 4;   // PRMT: T2 words
    uint2 *tab2 = reinterpret_cast<uint2 *>(smem);                     // GF(4): masks
    uint32_t *tabm = smem;                                             // GF(2): masks

    for (int i = 0; i < p.N; i++) {
        const int ii = i % kEncNI;
        if (ii == 0) {
            // resolve the coefficients of packets i .. i+NI-1 to their tables
            __syncthreads();
            const int ni = min(kEncNI, p.N - i);
            const int total = p.gens_per_cta * kEncNI * KT;
            for (int e = threadIdx.x; e < total; e += blockDim.x) {
                const int kk = e % KT;
                const int ie = (e / KT) % kEncNI;
                const int ge = e / (KT * kEncNI);
                uint32_t c = 0;
                if (ge < ngen && ie < ni && kk < kc)
                    c = p.C[((g_first + ge) * (size_t)p.N + (size_t)(i + ie)) * p.K + (k0 + kk)] &
                        (uint32_t)p.qmask;
                const uint32_t *t = p.tabs + (size_t)c * 8u;
                if (F == 256 || F == 16) {
                    tab4[e] = make_uint4(__ldg(t + 0), __ldg(t + 1), __ldg(t + 2), __ldg(t + 3));
                    tab1[e] = __ldg(t + 4);
                } else if (F == 4) {
                    tab2[e] = make_uint2(__ldg(t + 5), __ldg(t + 6));
                } else {
                    tabm[e] = __ldg(t + 5);
                }
            }
            __syncthreads();
        }
        if (!active) continue;

        // prefetch the next source packet's words
        if (i + 1 < p.N) {
            const uint8_t *An = Ag + (size_t)(i + 1) * p.M;
#pragma unroll
            for (int w = 0; w < W; w++) {
                const size_t wd = word0 + (size_t)w * 32u;
                nxt[w] = wd < p.Mw ? ld_word<BYTEWISE>(An, wd) : 0u;
            }
        }

        const int ebase = (gl * kEncNI + ii) * KT;
        if (F == 256 || F == 16) {
            Sel s[W];
#pragma unroll
            for (int w = 0; w < W; w++) s[w] = make_sel(cur[w]);
#pragma unroll
            for (int k = 0; k < KT; k++) {
                const uint4 t = tab4[ebase + k];
                PrmtTab T;
                T.t0lo = t.x; T.t0hi = t.y; T.t1lo = t.z; T.t1hi = t.w; T.t2 = tab1[ebase + k];
#pragma unroll
                for (int w = 0; w < W; w++) acc[k][w] ^= lookup_perm(T, s[w]);
            }
        } else if (F == 4) {
            uint32_t xa[W];
#pragma unroll
            for (int w = 0; w < W; w++) xa[w] = gf4_xtime(cur[w]);
#pragma unroll
            for (int k = 0; k < KT; k++) {
                const uint2 m = tab2[ebase + k];
#pragma unroll
                for (int w = 0; w < W; w++) acc[k][w] ^= (cur[w] & m.x) ^ (xa[w] & m.y);
            }
        } else {
#pragma unroll
            for (int k = 0; k < KT; k++) {
                const uint32_t m = tabm[ebase + k];
#pragma unroll
                for (int w = 0; w < W; w++) acc[k][w] ^= cur[w] & m;
            }
        }
#pragma unroll
        for (int w = 0; w < W; w++) cur[w] = nxt[w];
    }

    if (!active) return;
    uint8_t *Bg = p.B + g * (size_t)p.K * p.M;
#pragma unroll
    for (int k = 0; k < KT; k++) {
        if (k < kc) {
            uint8_t *row = Bg + (size_t)(k0 + k) * p.M;
#pragma unroll
            for (int w = 0; w < W; w++) {
                const size_t wd = word0 + (size_t)w * 32u;
                if (wd < p.Mw) {
                    const uint32_t v = (F == 256 || F == 16) ? unperm(acc[k][w]) : acc[k][w];
                    st_word<BYTEWISE>(row, wd, v);
                }
            }
        }
    }
}

}  // namespace gfr
