// encode_kernels.cuh -- batched RLNC encode B = A C over F_q (Eq. 2,
// PAPER.md:84-88), one kernel family per field.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]
//
// Work decomposition:
//   * a warp owns one generation g and a span of 32*W packet words (word =
//     4 bytes; lane l holds words span0 + w*32 + l, w < W, so every warp
//     access is a contiguous 128-byte line) -- the coefficients a warp needs
//     are therefore warp-uniform and every table read is a broadcast;
//   * a CTA owns KT coded packets k0 .. k0+KT-1 and either several whole
//     generations (short packets, e.g. M = 1500) or 8 spans of one generation
//     (long packets); the KT index varies fastest over the grid so the CTAs
//     that re-read the same A tile run together and hit L2;
//   * source words stream HBM -> shared memory through a per-thread ring of
//     S cp.async stages (each thread copies and later reads only its own
//     words, so no barrier guards the ring); each source word is loaded once
//     per CTA and reused for all KT outputs, and its coefficient-independent
//     preparation (PRMT selectors, bit planes) is amortised over KT;
//   * the coefficients of the current chunk of NI source packets are resolved
//     to compact per-field table entries in shared memory;
//   * accumulators (KT x W words) live in registers for the whole i loop and
//     B is written once (overwrite semantics, reading X8).
//
// BYTEWISE = true is the generic path for packets whose length is not a
// multiple of 4 or whose rows are not 4-byte aligned: a "word" is then a
// single byte zero-extended into a 32-bit register, which every field engine
// handles unchanged (a byte in lane 0 is a valid packed word); it loads
// straight from global memory.
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kEncNI = 16;   // source packets per table chunk

struct EncodeParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    const uint32_t *tabs;     // device table of tables, 16 words per coefficient
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

// ---- per-field inner products -------------------------------------------
// Two ways to form c * x on a 32-bit word of packed field elements:
//  * byte-permute lookups (PRMT, ALU pipe) -- the paper's shuffle, Alg. 1;
//  * the paper's imul (Alg. 2): isolate bit plane j of
//    every w-bit slot, multiply by the scalar pow[c][j] (IMAD, FMA pipe;
//    carry-free because each isolated bit contributes pow << slot_base with
//    pow < 2^w, reading X7), XOR the planes.
// The ALU pipe binds PRMT/LOP3 work, so fields split bit planes / outputs
// between the two pipes.  PRMT results come out
// in byte order [b0,b2,b1,b3]; imul planes are taken from the same permuted
// word so both agree, and the accumulator is un-permuted once at the end.
//
// Table entry words in the global table of tables (tables.cpp), per c:
//   0-3 T0lo,T0hi,T1lo,T1hi  4 T2  5 M0  6 M1  7 0  8-15 pow[c][0..7]
// Each engine keeps EW words per (i, k) in shared memory, chosen by the
// path output k takes (fill_entry).

template <int F, int KT> struct Engine;

// GF(256): bits 0-5 through two PRMT tables, bits 6-7 through two IMADs.
// Per (k, word): 2 PRMT + 2 LOP3 (ALU) + 2 IMAD (FMA).
template <int KT> struct Engine<256, KT> {
    static constexpr bool kPermuted = true;
    static constexpr int EW = 8;
    struct Word { uint32_t s0, s1, b6, b7; };
    __device__ __forceinline__ static void fill_entry(uint32_t *dst, const uint32_t *t, int)
    {
        reinterpret_cast<uint4 *>(dst)[0] = make_uint4(t[0], t[1], t[2], t[3]);
        reinterpret_cast<uint4 *>(dst)[1] = make_uint4(t[14], t[15], 0u, 0u);
    }
    __device__ __forceinline__ static Word prep(uint32_t x)
    {
        const uint32_t xp = prmt(x, x, 0x3120u);
        const uint32_t t0 = x & 0x07070707u;
        const uint32_t t1 = mul_hi(x, 1u << 29) & 0x07070707u;
        Word r;
        r.s0 = mad_hi(t0, 1u << 20, t0);
        r.s1 = mad_hi(t1, 1u << 20, t1);
        r.b6 = mul_hi(xp, 1u << 26) & 0x01010101u;
        r.b7 = mul_hi(xp, 1u << 25) & 0x01010101u;
        return r;
    }
    template <int W>
    __device__ __forceinline__ static void apply(uint32_t (&acc)[KT][W], const Word (&wd)[W],
                                                 const uint32_t *ent)
    {
#pragma unroll
        for (int k = 0; k < KT; k++) {
            const uint4 t = reinterpret_cast<const uint4 *>(ent + k * EW)[0];
            const uint2 p = reinterpret_cast<const uint2 *>(ent + k * EW)[2];
#pragma unroll
            for (int w = 0; w < W; w++) {
                uint32_t a = acc[k][w] ^ prmt(t.x, t.y, wd[w].s0) ^ prmt(t.z, t.w, wd[w].s1);
                acc[k][w] = a ^ (wd[w].b6 * p.x) ^ (wd[w].b7 * p.y);
            }
        }
    }
};

// GF(16): some outputs through 3 PRMT + 2 LOP3 (ALU 5), the others through
// 4 nibble-plane IMADs + 2 LOP3 (ALU 2, FMA 4); 5 of every 7 on IMAD
// balances the pipes at ~2.9 ops per (k, word) instead of 5.
template <int KT> struct Engine<16, KT> {
    static constexpr bool kPermuted = true;
    static constexpr int EW = 8;
    static constexpr int kImul = (KT * 5 + 3) / 7;
    struct Word { uint32_t s0, s1, s2, n0, n1, n2, n3; };
    __device__ __forceinline__ static void fill_entry(uint32_t *dst, const uint32_t *t, int k)
    {
        if (k < kImul) {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(t[8], t[9], t[10], t[11]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(0u, 0u, 0u, 0u);
        } else {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(t[0], t[1], t[2], t[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(t[4], 0u, 0u, 0u);
        }
    }
    __device__ __forceinline__ static Word prep(uint32_t x)
    {
        const uint32_t xp = prmt(x, x, 0x3120u);
        Word r;
        const Sel s = make_sel(x);
        r.s0 = s.s0; r.s1 = s.s1; r.s2 = s.s2;
        r.n0 = xp & 0x11111111u;
        r.n1 = mul_hi(xp, 1u << 31) & 0x11111111u;
        r.n2 = mul_hi(xp, 1u << 30) & 0x11111111u;
        r.n3 = mul_hi(xp, 1u << 29) & 0x11111111u;
        return r;
    }
    template <int W>
    __device__ __forceinline__ static void apply(uint32_t (&acc)[KT][W], const Word (&wd)[W],
                                                 const uint32_t *ent)
    {
#pragma unroll
        for (int k = 0; k < KT; k++) {
            const uint4 t = reinterpret_cast<const uint4 *>(ent + k * EW)[0];
            if (k < kImul) {
#pragma unroll
                for (int w = 0; w < W; w++) {
                    uint32_t a = acc[k][w] ^ (wd[w].n0 * t.x) ^ (wd[w].n1 * t.y);
                    acc[k][w] = a ^ (wd[w].n2 * t.z) ^ (wd[w].n3 * t.w);
                }
            } else {
                const uint32_t t2 = ent[k * EW + 4];
#pragma unroll
                for (int w = 0; w < W; w++) {
                    uint32_t a = acc[k][w] ^ prmt(t.x, t.y, wd[w].s0) ^ prmt(t.z, t.w, wd[w].s1);
                    acc[k][w] = a ^ prmt(t2, t2, wd[w].s2);
                }
            }
        }
    }
};

// GF(4): bit planes, x * (a1 x + a0) = (a0 + a1) x + a1.  Masked form
// c0*a ^ c1*(x a) costs 2 LOP3; imul form (a & 0x55)*c ^ ((a>>1) & 0x55)*(x c)
// costs 2 IMAD + 1 LOP3; 2 of every 3 outputs on IMAD -> ~1.33 per pipe.
template <int KT> struct Engine<4, KT> {
    static constexpr bool kPermuted = false;
    static constexpr int EW = 2;
    static constexpr int kImul = (KT * 2 + 1) / 3;
    struct Word { uint32_t a, xa, b0, b1; };
    __device__ __forceinline__ static void fill_entry(uint32_t *dst, const uint32_t *t, int k)
    {
        reinterpret_cast<uint2 *>(dst)[0] = k < kImul ? make_uint2(t[8], t[9]) : make_uint2(t[5], t[6]);
    }
    __device__ __forceinline__ static Word prep(uint32_t x)
    {
        Word r;
        r.a = x;
        r.xa = gf4_xtime(x);
        r.b0 = x & 0x55555555u;
        r.b1 = mul_hi(x, 1u << 31) & 0x55555555u;
        return r;
    }
    template <int W>
    __device__ __forceinline__ static void apply(uint32_t (&acc)[KT][W], const Word (&wd)[W],
                                                 const uint32_t *ent)
    {
#pragma unroll
        for (int k = 0; k < KT; k += 2) {
            uint4 t;                                                            // outputs k, k+1
            if (KT >= 2) t = reinterpret_cast<const uint4 *>(ent + k * EW)[0];
            else t = make_uint4(ent[0], ent[1], 0u, 0u);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int kk = k + h;
                if (kk >= KT) break;
                const uint32_t u0 = h ? t.z : t.x, u1 = h ? t.w : t.y;
#pragma unroll
                for (int w = 0; w < W; w++) {
                    if (kk < kImul) acc[kk][w] ^= (wd[w].b0 * u0) ^ (wd[w].b1 * u1);
                    else acc[kk][w] ^= (wd[w].a & u0) ^ (wd[w].xa & u1);
                }
            }
        }
    }
};

// GF(2): acc ^= a & mask(c): one LOP3 per (k, word); masks of 4 outputs per
// shared-memory load.
template <int KT> struct Engine<2, KT> {
    static constexpr bool kPermuted = false;
    static constexpr int EW = 1;
    struct Word { uint32_t a; };
    __device__ __forceinline__ static void fill_entry(uint32_t *dst, const uint32_t *t, int)
    {
        dst[0] = t[5];
    }
    __device__ __forceinline__ static Word prep(uint32_t x) { return Word{x}; }
    template <int W>
    __device__ __forceinline__ static void apply(uint32_t (&acc)[KT][W], const Word (&wd)[W],
                                                 const uint32_t *ent)
    {
#pragma unroll
        for (int k = 0; k < KT; k += 4) {
            uint4 m4;
            if (KT >= 4) m4 = reinterpret_cast<const uint4 *>(ent + k)[0];
            else m4 = make_uint4(ent[0], KT > 1 ? ent[1] : 0u, 0u, 0u);
            const uint32_t m[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
            for (int h = 0; h < 4; h++) {
                if (k + h >= KT) break;
#pragma unroll
                for (int w = 0; w < W; w++) acc[k + h][w] ^= wd[w].a & m[h];
            }
        }
    }
};

template <int F>
__host__ __device__ constexpr int enc_stages() { return F >= 16 ? 8 : 12; }

template <int F, int KT>
__host__ __device__ constexpr size_t enc_table_bytes_per_gen()
{
    return (size_t)kEncNI * KT * Engine<F, KT>::EW * 4u;
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

__device__ __forceinline__ void cp_async4(uint32_t smem_addr, const void *gptr, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;"
                 :: "r"(smem_addr), "l"(gptr), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

// S: cp.async ring depth (source packets in flight per thread)
template <int F, int W, int KT, int S, bool BYTEWISE>
__global__ void __launch_bounds__(256) encode_kernel(EncodeParams p)
{
    using E = Engine<F, KT>;
    extern __shared__ __align__(16) uint32_t smem[];
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

    uint32_t *tab = smem;                                                  // [gl][NI][KT][EW]
    uint32_t *ring = smem + (size_t)p.gens_per_cta * kEncNI * KT * E::EW;  // [S][W][blockDim]
    const uint8_t *Ag = p.A + (active ? g : 0) * (size_t)p.N * p.M;
    bool wvalid[W];
#pragma unroll
    for (int w = 0; w < W; w++) wvalid[w] = active && (word0 + (size_t)w * 32u) < p.Mw;

    // ---- source staging: cp.async ring (word path) or register prefetch (bytes)
    const uint32_t ring_base = (uint32_t)__cvta_generic_to_shared(ring) + threadIdx.x * 4u;
    auto issue = [&](int i) {
        const uint32_t slot = (uint32_t)(i % S) * W;
        const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)i * p.M);
#pragma unroll
        for (int w = 0; w < W; w++) {
            const size_t wd = word0 + (size_t)w * 32u;
            cp_async4(ring_base + (slot + w) * blockDim.x * 4u, wvalid[w] ? row + wd : row, wvalid[w]);
        }
    };
    uint32_t cur[W], nxt[W];
    if constexpr (BYTEWISE) {
#pragma unroll
        for (int w = 0; w < W; w++) cur[w] = wvalid[w] ? ld_word<true>(Ag, word0 + (size_t)w * 32u) : 0u;
    } else {
#pragma unroll
        for (int s = 0; s < S - 1; s++) {
            if (active && s < p.N) issue(s);
            cp_async_commit();
        }
    }

    for (int i = 0; i < p.N; i++) {
        const int ii = i % kEncNI;
        if (ii == 0) {
            // resolve the coefficients of packets i .. i+NI-1 to table entries
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
                E::fill_entry(tab + (size_t)e * E::EW, p.tabs + (size_t)c * 16u, kk);
            }
            __syncthreads();
        }
        if constexpr (BYTEWISE) {
            if (!active) continue;
            if (i + 1 < p.N) {
                const uint8_t *An = Ag + (size_t)(i + 1) * p.M;
#pragma unroll
                for (int w = 0; w < W; w++) nxt[w] = wvalid[w] ? ld_word<true>(An, word0 + (size_t)w * 32u) : 0u;
            }
        } else {
            if (active && i + S - 1 < p.N) issue(i + S - 1);
            cp_async_commit();
            cp_async_wait<S - 1>();
            if (!active) continue;
            const uint32_t *slot = ring + (size_t)(i % S) * W * blockDim.x + threadIdx.x;
#pragma unroll
            for (int w = 0; w < W; w++) cur[w] = slot[(size_t)w * blockDim.x];
        }

        typename E::Word wd[W];
#pragma unroll
        for (int w = 0; w < W; w++) wd[w] = E::prep(cur[w]);
        E::template apply<W>(acc, wd, tab + (size_t)(gl * kEncNI + ii) * KT * E::EW);

        if constexpr (BYTEWISE) {
#pragma unroll
            for (int w = 0; w < W; w++) cur[w] = nxt[w];
        }
    }
    if constexpr (!BYTEWISE) cp_async_wait<0>();

    if (!active) return;
    uint8_t *Bg = p.B + g * (size_t)p.K * p.M;
#pragma unroll
    for (int k = 0; k < KT; k++) {
        if (k < kc) {
            uint8_t *row = Bg + (size_t)(k0 + k) * p.M;
#pragma unroll
            for (int w = 0; w < W; w++) {
                if (wvalid[w]) {
                    const uint32_t v = E::kPermuted ? unperm(acc[k][w]) : acc[k][w];
                    st_word<BYTEWISE>(row, word0 + (size_t)w * 32u, v);
                }
            }
        }
    }
}

}  // namespace gfr
