// encode_prow.cuh -- batched RLNC encode through per-source "product rows":
// one shared-memory row per possible source BYTE value holding that byte's
// products with all coded-packet coefficients.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// The paper multiplies a region by one coefficient with split lookup tables
// indexed by source nibbles (Alg. 1).  Encode multiplies
// each source byte by K coefficients, so here the table is indexed by the
// whole source byte and returns K products at once:
//     P_i[a][k] = C[g][i][k] * a          a = 0..255, k in the CTA's 64
// (for GF(16)/GF(4)/GF(2) `*` is the packed product of every w-bit slot of the
// byte, so one byte-indexed row serves every field).  One 16-byte shared-
// memory load returns 16 finished products (16 byte-madds), against 4 bytes
// per load and two loads per GF(256) product for the nibble-table layouts
// (encode_lanek.cuh): the LSU pipe (128 B/clk/SM) then delivers 128
// byte-madds/clk/SM.
//
// Layout and conflict freedom.  A "group" is S = 4 source packets; its table
// is 256 rows x 256 B = 64 KiB: row a = [P_{4s}[a] | P_{4s+1}[a] | P_{4s+2}[a]
// | P_{4s+3}[a]], 64 B (= 64 coded packets) each.  Because a row spans two
// full bank sweeps, the bank of a 16-B chunk depends only on (source s mod 2,
// chunk kc) and never on the data byte a.  The 8 lanes of a quarter-warp (one
// LDS.128 wavefront) are 2 words x 4 chunks and the two words read sources of
// opposite parity (lane word jw reads source (jw + t) mod 4 at step t), so
// every LDS.128 is exactly 4 wavefronts for ANY data.
//
// Address generation: the two tables live at shared-window addresses 0x10000
// and 0x20000, so  addr = prmt(a_word, off, 0x76j4)  = [off.b0 = chunk offset,
// a_word.byte j = row, off.b2 = table] is one PRMT per 16-byte gather.
//
// Table build (per group, all 512 threads, overlapped with the previous
// group's gathers: double-buffered tables, one __syncthreads per group):
//   * basis rows P_i[2^b] (b < 8) from C by the packed xtime chain
//     (GF(2)-linearity: P[a] = XOR_{b in a} P[2^b]), staged one group ahead;
//   * thread (chunk, hi) writes rows hi*8 .. hi*8+7 in Gray-code order, one
//     16-byte XOR per row.
// Build traffic per group: 64 KiB of stores against TW * 4 * 64 B... gathers,
// i.e. 256 / (4 TW) of the gather traffic (17% for M = 1500).
//
// Work split: CTA = (generation, 64 coded packets, tile of TW words); lane =
// (word, 16-coefficient chunk); R words per lane (48 / 64 accumulator
// registers).  Source words are prefetched one group ahead straight from
// global memory into registers (no staging).  Epilogue: 4x4 byte transpose
// (8 PRMT) per 16 accumulator bytes, 4-byte stores (full 32-B sectors).
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kPrThreads = 512;
constexpr int kPrKC = 64;                   // coded packets per CTA
constexpr int kPrS = 4;                     // source packets per group (table)
constexpr uint32_t kPrTable0 = 0x10000u;    // shared-window address of table 0 (table 1 at 0x20000)
constexpr int kPrBasisBytes = 8 * 256;      // basis rows of one group

template <int R> struct PrGeom {
    static constexpr int WPW = 8;                       // words per warp per round
    static constexpr int TW = R * (kPrThreads / 32) * WPW;   // words per tile
};

struct ProwParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    size_t M;          // bytes per packet (multiple of 4)
    uint32_t Mw;       // words per packet
    int N, K;
    int NG;            // groups: ceil(N / 4)
    int tiles;         // word tiles per packet
    int k_tiles;       // ceil(K / 64)
    uint32_t qmask4;   // (q - 1) replicated in every byte
};

// x * v for packed elements (every w-bit slot of every byte, elements < q)
template <int F> __device__ __forceinline__ uint32_t pr_xtime(uint32_t a)
{
    if constexpr (F == 256) return ((a << 1) & 0xFEFEFEFEu) ^ (((a >> 7) & 0x01010101u) * 0x1Bu);
    else if constexpr (F == 16) return ((a << 1) & 0xEEEEEEEEu) ^ (((a >> 3) & 0x11111111u) * 3u);
    else if constexpr (F == 4) return gf4_xtime(a);
    else return a;
}

// P[2^b] for 4 coefficients c (one per byte, c < q): slot j = b / w of each
// byte holds c * x^(b mod w) -- the packed product of c with the byte 1 << b.
template <int F> __device__ __forceinline__ uint32_t pr_basis(uint32_t c, int b)
{
    constexpr int w = F == 256 ? 8 : F == 16 ? 4 : F == 4 ? 2 : 1;
    const int j = b / w, e = b - j * w;
    uint32_t v = c;
#pragma unroll
    for (int u = 0; u < w - 1; u++) {
        const uint32_t nv = pr_xtime<F>(v);
        v = u < e ? nv : v;
    }
    return v << (j * w);
}

__device__ __forceinline__ void sts128(uint32_t a, uint4 v)
{
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t u4c(const uint4 &v, int q)
{
    return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ void xor4(uint4 &a, const uint4 &b)
{
    a.x ^= b.x; a.y ^= b.y; a.z ^= b.z; a.w ^= b.w;
}

template <int F, int R>
__global__ void __launch_bounds__(kPrThreads, 1) encode_prow_kernel(ProwParams p)
{
    using G = PrGeom<R>;
    constexpr int TW = G::TW;
    extern __shared__ __align__(16) uint8_t pr_smem[];
    const int NP = p.NG * kPrS;                                // padded source count
    uint8_t *Cs = pr_smem;                                       // [NP][64] coefficients (masked)
    const uint32_t bas_s = (uint32_t)__cvta_generic_to_shared(pr_smem) + (uint32_t)NP * kPrKC;   // [2][8][256]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t bid = blockIdx.x;
    const int kt = (int)(bid % (size_t)p.k_tiles);
    const size_t rest = bid / (size_t)p.k_tiles;
    const int tile = (int)(rest % (size_t)p.tiles);
    const size_t g = rest / (size_t)p.tiles;
    const int k0 = kt * kPrKC;
    const uint32_t w0 = (uint32_t)tile * TW;
    const uint8_t *Ag = p.A + g * (size_t)p.N * p.M;

    // ---- gather-lane geometry
    const int qw = lane >> 3, ql = lane & 7;
    const int jw = ql >> 2, kc = ql & 3;
    uint32_t wd[R];
    bool wv[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        wd[r] = w0 + (uint32_t)(r * (kPrThreads / 32 * 8) + warp * 8 + qw * 2 + jw);
        wv[r] = wd[r] < p.Mw;
    }
    uint32_t areg[R][kPrS];
    auto load_a = [&](int grp) {
#pragma unroll
        for (int t = 0; t < kPrS; t++) {
            const int i = grp * kPrS + ((jw + t) & 3);
            const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
#pragma unroll
            for (int r = 0; r < R; r++) areg[r][t] = (wv[r] && i < p.N) ? __ldg(row + wd[r]) : 0u;
        }
    };
    load_a(0);

    // ---- coefficients of this CTA's 64 coded packets, zero past N / K
    {
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        for (int e = tid; e < NP * kPrKC; e += kPrThreads) {
            const int i = e >> 6, kk = e & 63;
            Cs[e] = (i < p.N && k0 + kk < p.K) ? (uint8_t)(Cg[(size_t)i * p.K + k0 + kk] & p.qmask4) : (uint8_t)0;
        }
    }
    __syncthreads();

    // basis rows of group grp into basis buffer buf: thread = (bit b, 16-B
    // chunk c16, word wq), 512 threads, one coefficient word each
    auto basis = [&](int grp, int buf) {
        const int wq = tid & 3, c16 = (tid >> 2) & 15, b = tid >> 6;
        const uint32_t c =
            *reinterpret_cast<const uint32_t *>(Cs + (grp * kPrS + (c16 >> 2)) * kPrKC + (c16 & 3) * 16 + wq * 4);
        const uint32_t v = pr_basis<F>(c, b);
        asm volatile("st.shared.u32 [%0], %1;" :: "r"(bas_s + buf * kPrBasisBytes + b * 256 + c16 * 16 + wq * 4),
                     "r"(v) : "memory");
    };
    // table of one group from basis buffer bbuf into table tbuf: thread
    // (chunk c16, hi) writes rows hi*8 .. hi*8+7 in Gray-code order
    auto build = [&](int bbuf, int tbuf) {
        const int c16 = tid & 15, hi = tid >> 4;
        const uint32_t bb = bas_s + bbuf * kPrBasisBytes + c16 * 16;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < 5; j++) {
            const uint4 b = lds128(bb + (3 + j) * 256);
            const uint32_t m = 0u - ((uint32_t)(hi >> j) & 1u);
            v.x ^= b.x & m; v.y ^= b.y & m; v.z ^= b.z & m; v.w ^= b.w & m;
        }
        uint4 bv[3];
#pragma unroll
        for (int b = 0; b < 3; b++) bv[b] = lds128(bb + b * 256);
        const uint32_t tb = kPrTable0 + (uint32_t)tbuf * 0x10000u + (uint32_t)hi * 8u * 256u + (uint32_t)c16 * 16u;
        sts128(tb + 0 * 256, v); xor4(v, bv[0]);
        sts128(tb + 1 * 256, v); xor4(v, bv[1]);
        sts128(tb + 3 * 256, v); xor4(v, bv[0]);
        sts128(tb + 2 * 256, v); xor4(v, bv[2]);
        sts128(tb + 6 * 256, v); xor4(v, bv[0]);
        sts128(tb + 7 * 256, v); xor4(v, bv[1]);
        sts128(tb + 5 * 256, v); xor4(v, bv[0]);
        sts128(tb + 4 * 256, v);
    };

    basis(0, 0);
    if (p.NG > 1) basis(1, 1);
    __syncthreads();
    build(0, 0);
    __syncthreads();

    uint4 acc[R][4];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);

#pragma unroll 1
    for (int it = 0; it < p.NG; it++) {
        if (it + 2 < p.NG) basis(it + 2, it & 1);
        if (it + 1 < p.NG) build((it + 1) & 1, (it + 1) & 1);
        const uint32_t tsel = (1u + (uint32_t)(it & 1)) << 16;
        const bool more = it + 1 < p.NG;
#pragma unroll
        for (int tp = 0; tp < kPrS; tp += 2) {
            // sources (jw + tp) and (jw + tp + 1) mod 4 of the group: two gathers per
            // accumulator, folded with one 3-input XOR
            const uint32_t off0 = tsel | (uint32_t)(((jw + tp) & 3) * 64 + kc * 16);
            const uint32_t off1 = tsel | (uint32_t)(((jw + tp + 1) & 3) * 64 + kc * 16);
            const int in0 = (it + 1) * kPrS + ((jw + tp) & 3), in1 = (it + 1) * kPrS + ((jw + tp + 1) & 3);
            const uint32_t *nrow0 = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(in0, p.N - 1) * p.M);
            const uint32_t *nrow1 = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(in1, p.N - 1) * p.M);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const uint32_t a0 = areg[r][tp], a1 = areg[r][tp + 1];
                if (more) {
                    areg[r][tp] = (wv[r] && in0 < p.N) ? __ldg(nrow0 + wd[r]) : 0u;
                    areg[r][tp + 1] = (wv[r] && in1 < p.N) ? __ldg(nrow1 + wd[r]) : 0u;
                }
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint4 v0 = lds128(prmt(a0, off0, 0x7604u | (j << 4)));
                    const uint4 v1 = lds128(prmt(a1, off1, 0x7604u | (j << 4)));
                    acc[r][j].x = xor3(acc[r][j].x, v0.x, v1.x);
                    acc[r][j].y = xor3(acc[r][j].y, v0.y, v1.y);
                    acc[r][j].z = xor3(acc[r][j].z, v0.z, v1.z);
                    acc[r][j].w = xor3(acc[r][j].w, v0.w, v1.w);
                }
            }
        }
        __syncthreads();
    }

    // ---- epilogue: acc[r][j] word q holds B[k0 + 16 kc + 4q + e][4 wd + j], e = byte;
    // transpose 4x4 bytes so that each output word is one coded packet's 4 bytes
#pragma unroll
    for (int r = 0; r < R; r++) {
        if (!wv[r]) continue;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t x0 = u4c(acc[r][0], q), x1 = u4c(acc[r][1], q);
            const uint32_t x2 = u4c(acc[r][2], q), x3 = u4c(acc[r][3], q);
            const uint32_t t0 = prmt(x0, x1, 0x5140u), t1 = prmt(x0, x1, 0x7362u);
            const uint32_t t2 = prmt(x2, x3, 0x5140u), t3 = prmt(x2, x3, 0x7362u);
            const uint32_t y[4] = {prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u), prmt(t1, t3, 0x5410u),
                                   prmt(t1, t3, 0x7632u)};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int k = k0 + kc * 16 + q * 4 + e;
                if (k < p.K)
                    reinterpret_cast<uint32_t *>(p.B + (g * (size_t)p.K + (size_t)k) * p.M)[wd[r]] = y[e];
            }
        }
    }
}

// dynamic shared memory: everything from the window base up to the end of
// table 1 (0x30000); the coefficient and basis buffers sit below table 0
__host__ __device__ constexpr size_t pr_low_bytes(int NG)
{
    return (size_t)NG * kPrS * kPrKC + 2 * (size_t)kPrBasisBytes;
}

}  // namespace gfr
