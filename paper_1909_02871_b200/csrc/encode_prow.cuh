// encode_prow.cuh -- batched RLNC encode through per-source "product rows":
// one shared-memory row per possible source BYTE value holding that byte's
// products with 64 coded-packet coefficients.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// The paper multiplies a region by one coefficient with split lookup tables
// indexed by source nibbles (Alg. 1).  Encode multiplies
// each source byte by K coefficients, so here the table is indexed by the
// whole source byte and returns 64 products at once:
//     P_i[a][k] = C[g][i][k] * a          a = 0..255, k in the CTA's 64
// (for GF(16)/GF(4)/GF(2) `*` is the packed product of every w-bit slot of the
// byte, so one byte-indexed row serves every field).  One 16-byte shared-
// memory load returns 16 finished products (16 byte-madds), against 4 bytes
// per load and two loads per GF(256) product for the nibble-table layouts
// (encode_lanek.cuh): the LSU pipe (128 B/clk/SM) delivers 128 byte-madds per
// clock and SM.
//
// Steps, tables and conflict freedom.  A "step" consumes 4 source packets.
// Its table is 256 rows x 256 B = 64 KiB, row a = [P_{4s}[a] | .. | P_{4s+3}[a]]
// (64 B each).  A row spans two full bank sweeps, so the bank of a 16-B chunk
// depends only on (source parity, coefficient chunk), never on the data byte
// a.  The 8 lanes of a quarter-warp (one LDS.128 wavefront) are 2 words x 4
// coefficient chunks, and the two words read sources of opposite parity
// (lane word jw reads source (jw + t) mod 4 at sub-step t): every LDS.128 is
// exactly 4 wavefronts for ANY data.  Address: prmt(a_word, col, 0x55j4) =
// a * 256 + col, plus the table base as the LDS immediate -- one PRMT per
// 16-byte gather.
//
// Pipeline.  Persistent CTAs (one per SM, 16 warps) walk a flattened sequence
// of steps over their tiles; three table buffers (at compile-time shared
// addresses, the loop is unrolled three times) and three basis buffers, with
// mbarrier rings instead of CTA-wide barriers.  Step s of every warp:
//   wait DONE(s-2), BASIS(s+1)  build table s+1          arrive BUILT(s+1)
//   wait BUILT(s)               basis rows of step s+3   arrive BASIS(s+3)
//   gather step s (LDS.128 product rows -> register accumulators)
//   write back when step s ends a tile (4x4 byte transpose)   arrive DONE(s)
// so a warp may run up to a step ahead of the slowest one.  Basis rows P[2^b]
// = C * x^b come from the packed xtime chain (one coefficient word per thread,
// loaded a step ahead, rows computed two steps ahead of their table); thread
// (chunk c16, hi) writes rows 8 hi .. 8 hi + 7 in Gray-code order, one 16-B
// XOR per row (P[a] = XOR_{b in a} P[2^b], GF(2)-linearity of the product).  Source words are prefetched one step
// ahead into registers straight from global memory.
// Build + basis traffic per step: 64 KiB + 16 KiB against 4 x 4 TW x 64 B of
// gathers (21% for TW = 384 words).
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kPrThreads = 512;
constexpr int kPrWarps = kPrThreads / 32;
constexpr int kPrKC = 64;                     // coded packets per CTA
constexpr int kPrS = 4;                       // source packets per step
constexpr uint32_t kPrBar = 0x0400u;          // mbarriers (6 x 8 B) at the dynamic window base
constexpr uint32_t kPrTab0 = 0x1000u;         // tables u = 0, 1, 2 at kPrTab0 + u * 0x10000
constexpr uint32_t kPrBasis = 0x31000u;       // basis rows: 3 buffers x 8 x 256 B
constexpr int kPrBasisBytes = 8 * 256;
constexpr uint32_t kPrSmemEnd = kPrBasis + 3 * kPrBasisBytes;

template <int R> struct PrGeom {
    static constexpr int WPW = 8;                              // words per warp per round
    static constexpr int TW = R * kPrWarps * WPW;              // words per tile
};

struct ProwParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    size_t M;          // bytes per packet (multiple of 4)
    uint32_t Mw;       // words per packet
    int N, K;
    int NS;            // steps per tile: ceil(N / 4)
    int tiles;         // word tiles per packet
    int k_tiles;       // ceil(K / 64)
    size_t ntiles;     // batch * tiles * k_tiles
    uint32_t qmask4;   // q - 1 in every byte
    int cword;         // coefficient rows can be read as 32-bit words
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
template <uint32_t OFF> __device__ __forceinline__ uint4 lds128_at(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+%5];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a), "n"(OFF));
    return v;
}
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t u4c(const uint4 &v, int q)
{
    return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}
__device__ __forceinline__ void xor4(uint4 &a, const uint4 &b)
{
    a.x ^= b.x; a.y ^= b.y; a.z ^= b.z; a.w ^= b.w;
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a)
{
    asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" :: "r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity)
{
    asm volatile("{ .reg .pred p;\n"
                 "PR_WAIT_%=:\n"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
                 "@!p bra PR_WAIT_%=;\n}" :: "r"(a), "r"(parity) : "memory");
}

// one work tile: generation g, coded packets k0 .. k0+63, words w0 .. w0+TW-1
struct PrTile {
    size_t g;
    int k0;
    uint32_t w0;
};

template <uint32_t V> struct PrU { static constexpr uint32_t value = V; };

template <int F, int R>
__global__ void __launch_bounds__(kPrThreads, 1) encode_prow_kernel(ProwParams p)
{
    constexpr int TW = PrGeom<R>::TW;
    // mbarrier rings (2 objects each, by step parity).  Phases: DONE(x), x >= 0,
    // on object x & 1 is phase x >> 1; BUILT(x), x >= 1, phase (x - 1) >> 1;
    // BASIS(x), x >= 3, phase (x - 3) >> 1 (table 0 and basis rows of steps 0..2
    // come from the prologue, ordered by __syncthreads).
    constexpr uint32_t kDone = kPrBar, kBuilt = kPrBar + 16, kBas = kPrBar + 32;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t ntile_cta = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t ntj = (uint32_t)ntile_cta;                 // tiles of this CTA
    const uint32_t total = ntj * (uint32_t)p.NS;             // steps of this CTA

    auto tile_of = [&](uint32_t j) {                          // j-th tile of this CTA
        const size_t t = blockIdx.x + (size_t)j * gridDim.x;
        PrTile r;
        const int kt = (int)(t % (size_t)p.k_tiles);
        const size_t rest = t / (size_t)p.k_tiles;
        r.w0 = (uint32_t)(rest % (size_t)p.tiles) * TW;
        r.g = rest / (size_t)p.tiles;
        r.k0 = kt * kPrKC;
        return r;
    };
    // step cursors (tile j, step st of the tile): divisions only at tile changes
    struct Cur {
        uint32_t j;
        int st;
        PrTile T;
    };
    auto cur_next = [&](Cur &c) {
        if (++c.st == p.NS) {
            c.st = 0;
            c.j++;
            c.T = tile_of(c.j);
        }
    };

    // ---- gather-lane geometry: quarter-warp = 2 words x 4 coefficient chunks
    const int qw = lane >> 3, ql = lane & 7;
    const int jw = ql >> 2, kc = ql & 3;
    uint32_t wofs[R];
#pragma unroll
    for (int r = 0; r < R; r++) wofs[r] = (uint32_t)(r * kPrWarps * 8 + warp * 8 + qw * 2 + jw);

    // source words of the cursor's step (4 sources x R words; sub-step t reads
    // source (jw + t) & 3), 0 past N / Mw
    auto load_a = [&](const Cur &c, uint32_t (&a)[R][kPrS]) {
        if (c.j >= ntj) return;
        const uint8_t *Ag = p.A + c.T.g * (size_t)p.N * p.M;
#pragma unroll
        for (int t = 0; t < kPrS; t++) {
            const int i = kPrS * c.st + ((jw + t) & 3);
            const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const uint32_t wd = c.T.w0 + wofs[r];
                a[r][t] = (i < p.N && wd < p.Mw) ? __ldg(row + wd) : 0u;
            }
        }
    };

    // basis thread geometry: word wq of 16-B chunk c16 (source c16 >> 2,
    // coefficients 16 (c16 & 3) + 4 wq .. +3), bit b
    const int bwq = tid & 3, bc16 = (tid >> 2) & 15, bb = tid >> 6;
    // raw coefficient word of the cursor's step (masked to F_q at use, so the
    // load is consumed a step later)
    auto load_c = [&](const Cur &cc) -> uint32_t {
        if (cc.j >= ntj) return 0u;
        const int i = kPrS * cc.st + (bc16 >> 2);
        if (i >= p.N) return 0u;
        const uint8_t *crow = p.C + (cc.T.g * (size_t)p.N + (size_t)i) * p.K;
        const int k = cc.T.k0 + 16 * (bc16 & 3) + 4 * bwq;
        if (p.cword) return k < p.K ? __ldg(reinterpret_cast<const uint32_t *>(crow + k)) : 0u;
        uint32_t c = 0;
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (k + e < p.K) c |= (uint32_t)__ldg(crow + k + e) << (8 * e);
        return c;
    };
    auto basis = [&](uint32_t s, uint32_t c, uint32_t buf) {  // buf = s % 3
        if (s < total)
            asm volatile("st.shared.u32 [%0], %1;" :: "r"(kPrBasis + buf * kPrBasisBytes + bb * 256 +
                                                         bc16 * 16 + bwq * 4),
                         "r"(pr_basis<F>(c & p.qmask4, bb)) : "memory");
    };
    // table of step s at shared address tab: thread (chunk c16, hi) -> rows 8 hi + Gray(0..7)
    auto build = [&](uint32_t s, uint32_t buf) {               // buf = s % 3
        if (s >= total) return;
        const int c16 = tid & 15, hi = tid >> 4;
        const uint32_t bsrc = kPrBasis + buf * kPrBasisBytes + c16 * 16;
        const uint32_t tab = kPrTab0 + buf * 0x10000u;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int j = 0; j < 5; j++) {
            const uint4 b = lds128(bsrc + (3 + j) * 256);
            const uint32_t m = 0u - ((uint32_t)(hi >> j) & 1u);
            v.x ^= b.x & m; v.y ^= b.y & m; v.z ^= b.z & m; v.w ^= b.w & m;
        }
        const uint4 b0 = lds128(bsrc), b1 = lds128(bsrc + 256), b2 = lds128(bsrc + 512);
        const uint32_t tb = tab + (uint32_t)hi * 8u * 256u + (uint32_t)c16 * 16u;
        sts128(tb + 0 * 256, v); xor4(v, b0);
        sts128(tb + 1 * 256, v); xor4(v, b1);
        sts128(tb + 3 * 256, v); xor4(v, b0);
        sts128(tb + 2 * 256, v); xor4(v, b2);
        sts128(tb + 6 * 256, v); xor4(v, b0);
        sts128(tb + 7 * 256, v); xor4(v, b1);
        sts128(tb + 5 * 256, v); xor4(v, b0);
        sts128(tb + 4 * 256, v);
    };

    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 6; b++) mbar_init(kPrBar + 8 * b, kPrWarps);
    }
    // ---- prologue: basis rows of steps 0..2, table 0, source words of step 0
    Cur ca;
    ca.j = 0; ca.st = 0; ca.T = tile_of(0);
    Cur cc = ca;
    uint32_t areg[R][kPrS];
    load_a(ca, areg);
    cur_next(ca);                                             // ca at step 1
    uint32_t creg;
    {
        const uint32_t c0 = load_c(cc); cur_next(cc);
        const uint32_t c1 = load_c(cc); cur_next(cc);
        const uint32_t c2 = load_c(cc); cur_next(cc);
        creg = load_c(cc); cur_next(cc);                      // step 3; cc at step 4
        basis(0, c0, 0);
        basis(1, c1, 1);
        basis(2, c2, 2);
    }
    __syncthreads();
    build(0, 0);
    __syncthreads();
    int st_g = 0;                                             // step-in-tile of the gather step
    uint32_t j_g = 0;

    uint4 acc[R][4];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);

    auto step = [&](uint32_t s, auto U) {
        constexpr uint32_t u = decltype(U)::value;            // table buffer of step s
        constexpr uint32_t un = (u + 1) % 3;                  // table buffer of step s + 1
        const uint32_t par = s & 1u;
        // ---- build table s + 1
        if (s >= 2) mbar_wait(kDone + par * 8u, ((s - 2) >> 1) & 1u);          // gathers of s-2 done
        if (s >= 2) mbar_wait(kBas + (par ^ 1u) * 8u, ((s - 2) >> 1) & 1u);   // basis rows of s+1
        build(s + 1, un);
        __syncwarp();
        if (lane == 0) mbar_arrive(kBuilt + (par ^ 1u) * 8u);
        // ---- basis rows of step s + 3 (their buffer held step s's, read by build(s))
        if (s >= 1) mbar_wait(kBuilt + par * 8u, ((s - 1) >> 1) & 1u);
        basis(s + 3, creg, u);
        creg = load_c(cc);                                    // step s + 4
        cur_next(cc);
        __syncwarp();
        if (lane == 0) mbar_arrive(kBas + (par ^ 1u) * 8u);
        // ---- gathers of step s
#pragma unroll
        for (int tp = 0; tp < kPrS; tp += 2) {
            const uint32_t col0 = (uint32_t)(((jw + tp) & 3) * 64 + kc * 16);
            const uint32_t col1 = (uint32_t)(((jw + tp + 1) & 3) * 64 + kc * 16);
#pragma unroll
            for (int r = 0; r < R; r++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint4 v0 =
                        lds128_at<kPrTab0 + u * 0x10000u>(prmt(areg[r][tp], col0, 0x5504u | (j << 4)));
                    const uint4 v1 =
                        lds128_at<kPrTab0 + u * 0x10000u>(prmt(areg[r][tp + 1], col1, 0x5504u | (j << 4)));
                    acc[r][j].x = xor3(acc[r][j].x, v0.x, v1.x);
                    acc[r][j].y = xor3(acc[r][j].y, v0.y, v1.y);
                    acc[r][j].z = xor3(acc[r][j].z, v0.z, v1.z);
                    acc[r][j].w = xor3(acc[r][j].w, v0.w, v1.w);
                }
            }
        }
        load_a(ca, areg);                                     // step s + 1
        cur_next(ca);
        if (++st_g == p.NS) {
            st_g = 0;
            // ---- write back the tile: acc[r][j] word q holds B[k0 + 16 kc + 4q + e][4 wd + j]
            // (e = byte); a 4x4 byte transpose makes each word one coded packet's 4 bytes
            const PrTile T = tile_of(j_g++);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const uint32_t wd = T.w0 + wofs[r];
                if (wd < p.Mw) {
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t x0 = u4c(acc[r][0], q), x1 = u4c(acc[r][1], q);
                        const uint32_t x2 = u4c(acc[r][2], q), x3 = u4c(acc[r][3], q);
                        const uint32_t t0 = prmt(x0, x1, 0x5140u), t1 = prmt(x0, x1, 0x7362u);
                        const uint32_t t2 = prmt(x2, x3, 0x5140u), t3 = prmt(x2, x3, 0x7362u);
                        const uint32_t y[4] = {prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u),
                                               prmt(t1, t3, 0x5410u), prmt(t1, t3, 0x7632u)};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int k = T.k0 + kc * 16 + q * 4 + e;
                            if (k < p.K)
                                reinterpret_cast<uint32_t *>(p.B + (T.g * (size_t)p.K + (size_t)k) * p.M)[wd] = y[e];
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(kDone + par * 8u);
    };

#pragma unroll 1
    for (uint32_t s = 0; s < total; s += 3) {
        step(s, PrU<0>{});
        if (s + 1 < total) step(s + 1, PrU<1>{});
        if (s + 2 < total) step(s + 2, PrU<2>{});
    }
}

}  // namespace gfr
