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
// Warp specialisation.  Persistent CTAs (one per SM) of 16 warps walk a
// flattened sequence of steps over their tiles (generation x 64 coded packets
// x 384 words):
//   * 12 gatherer warps (144 registers each, setmaxnreg): lane = (word,
//     16-coefficient chunk), 4 words per lane, 64 accumulator registers;
//     wait BUILT(s), gather step s from table s % 3, prefetch the source words
//     of step s+1 straight from global memory, write the tile back when s ends
//     it (4x4 byte transpose, 4-byte stores), arrive DONE(s);
//   * 4 producer warps (80 registers): wait DONE(s-3) (table buffer free);
//     thread (chunk c16, h) derives its chunk's basis rows P[2^b] = C * x^b
//     from the chunk's 16 coefficient bytes (packed xtime chain in registers,
//     coefficients prefetched a step ahead) and writes rows 32 h .. 32 h + 31
//     in Gray-code order, one 16-B XOR per row (P[a] = XOR_{b in a} P[2^b],
//     GF(2)-linearity of the product); arrive BUILT(s); one of them issues
//     an L2 bulk prefetch of the source rows of step s + 2.  (Computing the basis
//     once per chunk into shared memory and reading it back cost 4% of the
//     wavefronts and a producer barrier: C3 396.8 -> 409.7 GB/s without.)
// Three table buffers at compile-time shared addresses (the gatherer loop is
// unrolled three times so the table base is the LDS immediate), mbarrier
// rings of four objects; producers may run two steps ahead.
// Build traffic per step: 64 KiB against 4 x 4 x 384 x 64 B of gathers (17%).
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

constexpr int kPrThreads = 512;
constexpr int kPrGW = 12;                     // gatherer warps (warps 0..11)
constexpr int kPrPW = 4;                      // producer warps (warps 12..15, one warpgroup)
constexpr int kPrGRegs = 144, kPrPRegs = 80;  // setmaxnreg budgets: 12*32*144 + 4*32*80 = 65536 (80: no producer spill)
constexpr int kPrTW = 384;                    // words per tile
// Coded packets per CTA (KC = 64, or 32 for K <= 32): a table row (one source
// byte value) is 256 B = S sources x KC products, so a step covers S = 256 / KC
// source packets, a quarter-warp is WQ words x NKC 16-byte coefficient chunks
// (8 lanes on 8 distinct bank slots) and a lane holds R words (64 or 32
// accumulator registers).
template <int KC, int TW = kPrTW> struct PrCfg {
    static constexpr int S = 256 / KC;                         // sources per step (4 / 8)
    static constexpr int NKC = KC / 16;                        // 16-B chunks per source row (4 / 2)
    static constexpr int WQ = 8 / NKC;                         // words per quarter-warp (2 / 4)
    static constexpr int WPW = 4 * WQ;                         // words per warp per round
    static constexpr int R = TW / (kPrGW * WPW);               // words per gatherer lane (4 / 2; 4 for KC = 32, TW = 768)
    static_assert(R * kPrGW * WPW == TW, "tile geometry");
};
constexpr uint32_t kPrBar = 0x0400u;          // mbarriers: BUILT[4], DONE[4] at the dynamic window base
constexpr uint32_t kPrTab0 = 0x1000u;         // tables u = 0, 1, 2 at kPrTab0 + u * 0x10000
constexpr uint32_t kPrSmemEnd = kPrTab0 + 3 * 0x10000u;

struct ProwParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    size_t M;          // bytes per packet (multiple of 4)
    uint32_t Mw;       // words per packet
    int N, K;
    int NS;            // steps per tile: ceil(N / S)
    int tiles;         // word tiles per packet
    int k_tiles;       // ceil(K / KC)
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
__device__ __forceinline__ void nbar_sync_n(int id, int n)
{
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}

// one work tile: generation g, coded packets k0 .. k0+63, words w0 .. w0+TW-1
struct PrTile {
    size_t g;
    int k0;
    uint32_t w0;
};

template <uint32_t V> struct PrU { static constexpr uint32_t value = V; };

// TW: words per tile (384; 768 with 32 coded packets per CTA for long packets:
// a table then serves twice the gathers, halving the build share)
template <int F, int KC, int TW = kPrTW>
__global__ void __launch_bounds__(kPrThreads, 1) encode_prow_kernel(ProwParams p)
{
    using Cf = PrCfg<KC, TW>;
    constexpr int kPrS = Cf::S, NKC = Cf::NKC;
    // mbarrier rings, object x & 3 for step x: BUILT(x) (4 producer-warp
    // arrivals) is phase x >> 2; DONE(x) (12 gatherer-warp arrivals) is phase
    // (x + 4) >> 2, the virtual steps -4..-1 pre-arrived.
    constexpr uint32_t kBuilt = kPrBar, kDone = kPrBar + 32;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t ntile_cta = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t ntj = (uint32_t)ntile_cta;                 // tiles of this CTA
    const uint32_t total = ntj * (uint32_t)p.NS;             // steps of this CTA

    auto tile_of = [&](uint32_t j) {                          // j-th tile of this CTA
        const size_t t = blockIdx.x + (size_t)(j < ntj ? j : 0u) * gridDim.x;
        PrTile r;
        const int kt = (int)(t % (size_t)p.k_tiles);
        const size_t rest = t / (size_t)p.k_tiles;
        r.w0 = (uint32_t)(rest % (size_t)p.tiles) * TW;
        r.g = rest / (size_t)p.tiles;
        r.k0 = kt * KC;
        return r;
    };

    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 4; b++) {
            mbar_init(kBuilt + 8 * b, kPrPW);
            mbar_init(kDone + 8 * b, kPrGW);
        }
#pragma unroll
        for (int b = 0; b < 4; b++) mbar_arrive_n(kDone + 8 * b, kPrGW);   // DONE(-4 .. -1)
    }
    __syncthreads();

    if (warp >= kPrGW) {
        // ======================= producers: basis rows + tables
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(kPrPRegs));
        const int pt = tid - kPrGW * 32;                       // 0 .. 127
        // thread (chunk c16, row group h3): table rows 32 h3 .. 32 h3 + 31 of the
        // 16-byte chunk c16 = (source c16 / NKC, coefficient chunk c16 % NKC).
        // Each thread derives its chunk's 8 basis rows P[2^b] = C * x^b itself
        // from the 16 raw coefficient bytes (packed xtime chain in registers):
        // no shared-memory basis buffer, no producer barrier.
        const int c16 = pt & 15, h3 = pt >> 4;
        const int csrc = c16 / NKC, ckc = c16 % NKC;
        const bool c16ok = p.K % 16 == 0 && (reinterpret_cast<uintptr_t>(p.C) & 15u) == 0;
        // coefficient cursor: &C[g][S st + csrc][k0 + 16 ckc]
        uint32_t cj = 0;
        int cst = 0;
        const uint8_t *cptr = nullptr;
        int ck = 0;
        bool kok = false;
        auto setc = [&]() {
            const PrTile T = tile_of(cj);
            ck = T.k0 + 16 * ckc;
            cptr = p.C + (T.g * (size_t)p.N + (size_t)csrc) * p.K + ck;
            kok = cj < ntj && ck < p.K;
        };
        auto load_c = [&]() -> uint4 {                         // 16 raw coefficient bytes of the cursor's step
            uint4 c = make_uint4(0u, 0u, 0u, 0u);
            if (kok && kPrS * cst + csrc < p.N) {
                if (c16ok) {
                    c = __ldg(reinterpret_cast<const uint4 *>(cptr));
                } else {
                    uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int e = 0; e < 16; e++)
                        if (ck + e < p.K) wv[e >> 2] |= (uint32_t)__ldg(cptr + e) << (8 * (e & 3));
                    c = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
            }
            if (++cst == p.NS) {
                cst = 0;
                cj++;
                setc();
            } else {
                cptr += (size_t)kPrS * p.K;
            }
            return c;
        };
        auto build = [&](const uint4 craw, uint32_t tab) {
            constexpr int w = F == 256 ? 8 : F == 16 ? 4 : F == 4 ? 2 : 1;
            uint32_t bvw[5][4], vw[4];
#pragma unroll
            for (int q = 0; q < 4; q++) {
                // basis bit b of coefficient word q: slot b / w holds c * x^(b mod w)
                uint32_t xt[w];
                xt[0] = u4c(craw, q) & p.qmask4;
#pragma unroll
                for (int e = 1; e < w; e++) xt[e] = pr_xtime<F>(xt[e - 1]);
                uint32_t vq = 0u;
#pragma unroll
                for (int bb = 0; bb < 8; bb++) {
                    const uint32_t rb = xt[bb % w] << ((bb / w) * w);
                    if (bb < 5) bvw[bb][q] = rb;
                    else vq ^= rb & (0u - ((uint32_t)(h3 >> (bb - 5)) & 1u));   // rows 5..7 selected by h3
                }
                vw[q] = vq;
            }
            uint4 v = make_uint4(vw[0], vw[1], vw[2], vw[3]);
            uint4 bv[5];
#pragma unroll
            for (int j = 0; j < 5; j++) bv[j] = make_uint4(bvw[j][0], bvw[j][1], bvw[j][2], bvw[j][3]);
            const uint32_t tb = tab + (uint32_t)h3 * 32u * 256u + (uint32_t)c16 * 16u;
            sts128(tb, v);
#pragma unroll
            for (int n = 1; n < 32; n++) {
                const int flip = (n & 1) ? 0 : (n & 2) ? 1 : (n & 4) ? 2 : (n & 8) ? 3 : 4;   // Gray code: bit flipped at step n
                xor4(v, bv[flip]);
                sts128(tb + (uint32_t)(n ^ (n >> 1)) * 256u, v);
            }
        };

        // L2 prefetch of the gatherers' source rows: one bulk prefetch per
        // source row segment of step x + PD (the producers run up to three steps
        // ahead of the gatherers, whose per-lane loads then hit L2, not HBM)
        constexpr uint32_t PD = 2;
        auto prefetch_step = [&](uint32_t x) {
            const uint32_t j = x / (uint32_t)p.NS, st = x - j * (uint32_t)p.NS;
            if (j >= ntj) return;
            const PrTile T = tile_of(j);
            const uint32_t nw = min((uint32_t)TW, p.Mw - T.w0);
            const uint8_t *row0 = p.A + T.g * (size_t)p.N * p.M + 4 * (size_t)T.w0;
            if (st == 0) {                                      // a new tile: its coefficient block too
                const uintptr_t c = reinterpret_cast<uintptr_t>(p.C + T.g * (size_t)p.N * p.K);
                const uintptr_t c0 = c & ~(uintptr_t)15, c1 = (c + (uintptr_t)p.N * p.K + 15) & ~(uintptr_t)15;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(c0), "r"((uint32_t)(c1 - c0)) : "memory");
            }
#pragma unroll
            for (int t = 0; t < kPrS; t++) {
                const int i = kPrS * (int)st + t;
                if (i >= p.N) break;
                const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + (size_t)i * p.M);
                const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + 4 * (uintptr_t)nw + 15) & ~(uintptr_t)15;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
            }
        };
        if (pt == 0)
            for (uint32_t x = 1; x < PD; x++) prefetch_step(x);

        setc();
        uint4 creg = load_c();                                  // step 0
#pragma unroll 1
        for (uint32_t x = 0; x < total; x++) {                  // table of step x
            if (pt == 0) prefetch_step(x + PD);
            mbar_wait_sleepy(kDone + ((x - 3) & 3u) * 8u, ((x + 1) >> 2) & 1u);   // DONE(x-3): buffer free
            const uint4 c = creg;
            creg = load_c();                                    // step x + 1
            build(c, kPrTab0 + (x % 3u) * 0x10000u);
            __syncwarp();
            if (lane == 0) mbar_arrive(kBuilt + (x & 3u) * 8u);
        }
        return;
    }

    // ======================= gatherers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(kPrGRegs));
    constexpr int R = Cf::R;
    const int qw = lane >> 3, ql = lane & 7;
    const int jw = ql / NKC, kc = ql % NKC;
    const uint32_t wbase = (uint32_t)(warp * Cf::WPW + qw * Cf::WQ + jw);   // word r: wbase + kRW r
    constexpr uint32_t kRW = kPrGW * Cf::WPW;

    // source-word cursor: a = &A[g][4 st][w0 + wbase] (bytes), vmask bit r = word r valid
    uint32_t aj = 0;
    int ast = 0;
    const uint8_t *aptr = nullptr;
    uint32_t vmask = 0;
    auto seta = [&]() {
        const PrTile T = tile_of(aj);
        aptr = p.A + T.g * (size_t)p.N * p.M + 4 * (size_t)(T.w0 + wbase);
        vmask = 0;
#pragma unroll
        for (int r = 0; r < R; r++)
            if (aj < ntj && T.w0 + wbase + kRW * r < p.Mw) vmask |= 1u << r;
    };
    uint32_t areg[R][kPrS];
    // byte offset of sub-step t's source row within the step: ((jw + t) mod S) * M
    size_t soff[kPrS];
#pragma unroll
    for (int t = 0; t < kPrS; t++) soff[t] = (size_t)((jw + t) & (kPrS - 1)) * p.M;
    auto load_a = [&]() {                                      // the cursor's step, then advance
        const int nsrc = p.N - kPrS * ast;                     // sources of the step that exist
#pragma unroll
        for (int t = 0; t < kPrS; t++) {
            const bool iok = ((jw + t) & (kPrS - 1)) < nsrc;
            const uint32_t *row = reinterpret_cast<const uint32_t *>(aptr + soff[t]);
#pragma unroll
            for (int r = 0; r < R; r++) areg[r][t] = (iok && (vmask >> r & 1u)) ? __ldg(row + kRW * r) : 0u;
        }
        if (++ast == p.NS) {
            ast = 0;
            aj++;
            seta();
        } else {
            aptr += (size_t)kPrS * p.M;
        }
    };
    seta();
    uint32_t gmask = vmask;                                    // words of the gather tile that exist
    load_a();                                                  // step 0

    uint4 acc[R][4];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);
    int st_g = 0;                                              // step-in-tile of the gather step
    uint32_t j_g = 0;

    auto step = [&](uint32_t s, auto U) {
        constexpr uint32_t u = decltype(U)::value;             // table buffer of step s
        mbar_wait(kBuilt + (s & 3u) * 8u, (s >> 2) & 1u);
        // table column of sub-step t: source (jw + t) mod S, coefficient chunk kc
        uint32_t col[kPrS];
#pragma unroll
        for (int t = 0; t < kPrS; t++) col[t] = (uint32_t)(((jw + t) & (kPrS - 1)) * KC + kc * 16);
#pragma unroll
        for (int r = 0; r < R; r++) {
            if (!(gmask >> r & 1u)) continue;                  // past the packet end: no gathers (partial tiles)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t sel = 0x5504u | (j << 4);
#pragma unroll
                for (int t = 0; t < kPrS; t += 2) {
                    const uint4 v0 = lds128_at<kPrTab0 + u * 0x10000u>(prmt(areg[r][t], col[t], sel));
                    const uint4 v1 = lds128_at<kPrTab0 + u * 0x10000u>(prmt(areg[r][t + 1], col[t + 1], sel));
                    acc[r][j].x = xor3(acc[r][j].x, v0.x, v1.x);
                    acc[r][j].y = xor3(acc[r][j].y, v0.y, v1.y);
                    acc[r][j].z = xor3(acc[r][j].z, v0.z, v1.z);
                    acc[r][j].w = xor3(acc[r][j].w, v0.w, v1.w);
                }
            }
        }
        // table s is free once this warp's gathers are performed (release
        // semantics of the arrive); tell the producers before the next step's
        // source loads and a tile's write-back
        __syncwarp();
        if (lane == 0) mbar_arrive(kDone + (s & 3u) * 8u);
        load_a();                                              // step s + 1
        if (++st_g == p.NS) {
            st_g = 0;
            // ---- write back the tile: acc[r][j] word q holds B[k0 + 16 kc + 4q + e][4 wd + j]
            // (e = byte); a 4x4 byte transpose makes each word one coded packet's 4 bytes
            const PrTile T = tile_of(j_g++);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const uint32_t wd = T.w0 + wbase + kRW * r;
                if (wd < p.Mw) {
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t x0 = u4c(acc[r][0], q), x1 = u4c(acc[r][1], q);
                        const uint32_t x2 = u4c(acc[r][2], q), x3 = u4c(acc[r][3], q);
                        const uint32_t t0 = prmt(x0, x1, 0x5140u), t1 = prmt(x0, x1, 0x7362u);
                        const uint32_t t2 = prmt(x2, x3, 0x5140u), t3 = prmt(x2, x3, 0x7362u);
                        uint32_t y[4] = {prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u),
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
            const PrTile Tn = tile_of(j_g);                     // the next gather tile's words
            gmask = 0;
#pragma unroll
            for (int r = 0; r < R; r++)
                if (j_g < ntj && Tn.w0 + wbase + kRW * r < p.Mw) gmask |= 1u << r;
        }
    };

#pragma unroll 1
    for (uint32_t s = 0; s < total; s += 3) {
        step(s, PrU<0>{});
        if (s + 1 < total) step(s + 1, PrU<1>{});
        if (s + 2 < total) step(s + 2, PrU<2>{});
    }
}

}  // namespace gfr
