// encode_lanek2.cuh -- persistent, mbarrier-pipelined lane-k encode for the
// small fields (GF(2), GF(4)) with up to 32 coded packets (C5).
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Same arithmetic as encode_lanek.cuh -- a step of SG source packets (4 for
// GF(2), 2 for GF(4)) becomes, for every word w of the tile, a 16-row table of
// XOR combinations of four generator values (the paper's split-table idea,
// Alg. 1, with data and coefficient exchanged: a "four
// Russians" table over the coefficient bits), and lane k of a gatherer warp
// reads the row of ITS coefficients (one LDS per 32 products, <= 16 distinct
// rows in distinct banks: one wavefront) -- but organised for the memory-bound
// C5 shape, where each CTA of the one-shot kernel lived for only N/SG = 8 steps:
//   * persistent CTAs (one per SM, 32 warps) walk a flattened (tile, step)
//     sequence; tile = generation x 512 words;
//   * 16 producer warps: source words straight from global memory into
//     registers six steps ahead, 16-row table of step s into Q[s % 3], and
//     (warp 16) the per-lane row indices of step s into a small ring; arrive
//     FULL(s) after waiting DONE(s-3);
//   * 16 gatherer warps (lane = k, 32 words per lane): wait FULL(s), 32
//     gathers + XORs, arrive DONE(s); at a tile end each warp transposes its
//     32 x 32-word block through its own shared-memory scratch (no cross-warp
//     barrier) and writes 128-byte rows.
// mbarrier rings of four objects (producers may run three steps ahead).
#pragma once
#include <cstdint>

#include "encode_lanek.cuh"
#include "encode_prow.cuh"   // mbarrier helpers

namespace gfr {

constexpr int kL2GW = 16;                        // gatherer warps (0..15)
constexpr int kL2PW = 16;                        // producer warps (16..31)
constexpr int kL2Threads = 32 * (kL2GW + kL2PW);
constexpr int kL2TW = 32 * kL2GW;                // words per tile (512)
constexpr int kL2QS = kL2TW + 1;                 // Q row stride (odd: gathers conflict-free)
constexpr int kL2NQ = 3;                         // table buffers
constexpr int kL2QWords = 16 * kL2QS;
constexpr int kL2ScrS = 33;                      // epilogue scratch row stride (words)
constexpr int kL2BWords = kL2TW / (32 * kL2PW);  // words per producer thread per step (1)
constexpr int kL2D = 6;                          // source-word prefetch distance (steps)

struct Lk2Params {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    size_t M;          // bytes per packet (multiple of 4)
    uint32_t Mw;       // words per packet
    int N, K;          // K <= 32
    int NS;            // steps per tile: ceil(N / SG)
    int tiles;         // word tiles per packet
    size_t ntiles;     // batch * tiles
};

// shared memory: mbarriers | Q[3][16][QS] | row-index ring [3][32] | scratch[16][32][33]
constexpr size_t kL2OffQ = 64;
constexpr size_t kL2OffIdx = kL2OffQ + (size_t)kL2NQ * kL2QWords * 4;
constexpr size_t kL2OffScr = kL2OffIdx + (size_t)kL2NQ * 32;
constexpr size_t kL2Smem = kL2OffScr + (size_t)kL2GW * 32 * kL2ScrS * 4;

template <int F>
__global__ void __launch_bounds__(kL2Threads, 1) encode_lanek2_kernel(Lk2Params p)
{
    using L = LkField<F>;
    constexpr int SG = L::kSG;
    static_assert(F == 2 || F == 4, "small fields only");
    extern __shared__ __align__(16) uint8_t l2_smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(l2_smem);
    const uint32_t kFull = sbase, kDone = sbase + 32;        // 4 + 4 mbarriers
    uint32_t *Q = reinterpret_cast<uint32_t *>(l2_smem + kL2OffQ);
    uint8_t *idx = l2_smem + kL2OffIdx;
    uint32_t *scr = reinterpret_cast<uint32_t *>(l2_smem + kL2OffScr);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t ntile_cta = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t ntj = (uint32_t)ntile_cta;
    const uint32_t total = ntj * (uint32_t)p.NS;

    auto tile_g = [&](uint32_t j, uint32_t &w0) {           // generation and first word of the CTA's j-th tile
        const size_t t = blockIdx.x + (size_t)(j < ntj ? j : 0u) * gridDim.x;
        w0 = (uint32_t)(t % (size_t)p.tiles) * kL2TW;
        return t / (size_t)p.tiles;
    };

    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 4; b++) {
            mbar_init(kFull + 8 * b, kL2PW);
            mbar_init(kDone + 8 * b, kL2GW);
        }
#pragma unroll
        for (int b = 0; b < 4; b++) mbar_arrive_n(kDone + 8 * b, kL2GW);   // DONE(-4 .. -1)
    }
    __syncthreads();

    if (warp >= kL2GW) {
        // ======================= producers
        const int pt = tid - 32 * kL2GW;                       // 0 .. 32 * kL2PW - 1
        // source cursor
        uint32_t aj = 0, aw0 = 0;
        int ast = 0;
        size_t ag = tile_g(0, aw0);
        uint32_t ar[kL2D][kL2BWords][SG];
        auto load = [&](uint32_t (&a)[kL2BWords][SG]) {      // the cursor's step, then advance
            const bool live = aj < ntj;
            const uint8_t *Ag = p.A + ag * (size_t)p.N * p.M;
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = ast * SG + j;
                const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
#pragma unroll
                for (int u = 0; u < kL2BWords; u++) {
                    const uint32_t wd = aw0 + (uint32_t)pt + 32u * kL2PW * u;
                    a[u][j] = (live && i < p.N && wd < p.Mw) ? __ldg(row + wd) : 0u;
                }
            }
            if (++ast == p.NS) {
                ast = 0;
                aj++;
                ag = tile_g(aj, aw0);
            }
        };
        // coefficient-index cursor (warp 16 only): lane k's row index of each step
        uint32_t cj = 0, cw0 = 0;
        int cst = 0;
        size_t cg = tile_g(0, cw0);
        auto row_index = [&]() -> uint32_t {                  // the cursor's step, then advance
            uint8_t c[SG];
            const uint8_t *Cg = p.C + cg * (size_t)p.N * p.K;
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = cst * SG + j;
                c[j] = (cj < ntj && i < p.N && lane < p.K) ? __ldg(Cg + (size_t)i * p.K + lane) : (uint8_t)0;
            }
            if (++cst == p.NS) {
                cst = 0;
                cj++;
                cg = tile_g(cj, cw0);
            }
            return L::index(c);
        };
        auto pstep = [&](uint32_t s, uint32_t b, uint32_t (&a)[kL2BWords][SG]) {
            mbar_wait(kDone + ((s - 3) & 3u) * 8u, ((s + 1) >> 2) & 1u);   // DONE(s-3): buffer b free
            uint32_t *q = Q + b * kL2QWords;
#pragma unroll
            for (int u = 0; u < kL2BWords; u++) build_word<F, kL2QS>(q + pt + 32 * kL2PW * u, a[u]);
            if (warp == kL2GW) idx[b * 32 + lane] = (uint8_t)row_index();
            __syncwarp();
            if (lane == 0) mbar_arrive(kFull + (s & 3u) * 8u);
            load(a);                                           // step s + kL2D
        };
        // zero rows of every buffer (row index 0 = no source selected)
        for (int t = pt; t < kL2NQ * kL2QS; t += 32 * kL2PW) Q[(t / kL2QS) * kL2QWords + t % kL2QS] = 0u;
#pragma unroll
        for (int d = 0; d < kL2D; d++) load(ar[d]);
        static_assert(kL2D == 6 && kL2NQ == 3, "producer loop unrolled 6 = 2 x NQ");
#pragma unroll 1
        for (uint32_t s = 0; s < total; s += 6) {
            pstep(s, 0, ar[0]);
            if (s + 1 < total) pstep(s + 1, 1, ar[1]);
            if (s + 2 < total) pstep(s + 2, 2, ar[2]);
            if (s + 3 < total) pstep(s + 3, 0, ar[3]);
            if (s + 4 < total) pstep(s + 4, 1, ar[4]);
            if (s + 5 < total) pstep(s + 5, 2, ar[5]);
        }
        return;
    }

    // ======================= gatherers: lane = coded packet k, words 32 gw .. 32 gw + 31
    uint32_t *myscr = scr + warp * 32 * kL2ScrS;
    uint32_t acc[32];
#pragma unroll
    for (int w = 0; w < 32; w++) acc[w] = 0u;
    int st_g = 0;
    uint32_t j_g = 0;
    auto gstep = [&](uint32_t s, uint32_t b) {
        mbar_wait(kFull + (s & 3u) * 8u, (s >> 2) & 1u);
        const uint32_t r = idx[b * 32 + lane];
        const uint32_t *row = Q + b * kL2QWords + r * kL2QS + warp * 32;
#pragma unroll
        for (int w = 0; w < 32; w++) acc[w] ^= row[w];
        __syncwarp();
        if (lane == 0) mbar_arrive(kDone + (s & 3u) * 8u);
        if (++st_g == p.NS) {
            st_g = 0;
            // ---- write back: transpose the warp's 32 x 32-word block through its scratch
            uint32_t w0;
            const size_t g = tile_g(j_g++, w0);
#pragma unroll
            for (int w = 0; w < 32; w++) {
                myscr[lane * kL2ScrS + w] = acc[w];
                acc[w] = 0u;
            }
            __syncwarp();
            const uint32_t wd = w0 + (uint32_t)(warp * 32 + lane);
            if (wd < p.Mw) {
                uint32_t *Bg = reinterpret_cast<uint32_t *>(p.B + g * (size_t)p.K * p.M) + wd;
                for (int k = 0; k < p.K; k++) Bg[(size_t)k * p.Mw] = myscr[k * kL2ScrS + lane];
            }
            __syncwarp();
        }
    };
#pragma unroll 1
    for (uint32_t s = 0; s < total; s += 3) {
        gstep(s, 0);
        if (s + 1 < total) gstep(s + 1, 1);
        if (s + 2 < total) gstep(s + 2, 2);
    }
}

}  // namespace gfr
