// encode_lanek2.cuh -- persistent lane-k encode for the small fields (GF(2),
// GF(4)) with up to 32 coded packets (C5).
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Same arithmetic as encode_lanek.cuh -- a step of SG source packets (4 for
// GF(2), 2 for GF(4)) becomes, for every word w of the tile, a 16-row table of
// XOR combinations of four generator values (the paper's split-table idea,
// Alg. 1, with data and coefficient exchanged: a "four
// Russians" table over the coefficient bits), and lane k of a gatherer warp
// reads the row of ITS coefficients (one LDS per 32 products, <= 16 distinct
// rows in distinct banks: one wavefront).  The one-shot kernel's CTAs live for
// only N/SG = 8 steps on C5, so every CTA pays its start (first source loads,
// coefficient indices) and its write-back unoverlapped; here CTAs are
// persistent (two per SM) and walk a flattened (tile, step) sequence:
//   * 4 builder warps: source words straight from global memory into
//     registers three steps ahead (across tile boundaries), the 16-row table
//     of step s into Q[s % 3] and (first builder warp) the per-lane row
//     indices of step s into a 3-slot ring; named barriers FULL / EMPTY per
//     buffer hand the tables to the gatherers, as in the one-shot kernel;
//   * 8 gatherer warps (lane = k, 32 words per lane): 32 gathers + XORs per
//     step; at a tile end each warp transposes its 32 x 32-word block through
//     its own shared-memory scratch (no cross-warp barrier) and writes
//     128-byte rows, while the builders already fill the next tile's tables.
#pragma once
#include <cstdint>

#include "encode_lanek.cuh"

namespace gfr {

constexpr int kL2GW = 8;                         // gatherer warps (0..7)
constexpr int kL2BW = 4;                         // builder warps (8..11)
constexpr int kL2Threads = 32 * (kL2GW + kL2BW);
constexpr int kL2TW = 32 * kL2GW;                // words per tile (256)
constexpr int kL2QS = kL2TW + 1;                 // Q row stride (odd: gathers conflict-free)
constexpr int kL2NQ = 3;                         // table buffers
constexpr int kL2QWords = 16 * kL2QS;
constexpr int kL2ScrS = 33;                      // epilogue scratch row stride (words)
constexpr int kL2BWords = kL2TW / (32 * kL2BW);  // words per builder thread per step (2)

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

// shared memory: Q[3][16][QS] | row-index ring [3][32] | scratch[8][32][33]
constexpr size_t kL2OffIdx = (size_t)kL2NQ * kL2QWords * 4;
constexpr size_t kL2OffScr = kL2OffIdx + (size_t)kL2NQ * 32;
constexpr size_t kL2Smem = kL2OffScr + (size_t)kL2GW * 32 * kL2ScrS * 4;

template <int F>
__global__ void __launch_bounds__(kL2Threads, 2) encode_lanek2_kernel(Lk2Params p)
{
    using L = LkField<F>;
    constexpr int SG = L::kSG;
    static_assert(F == 2 || F == 4, "small fields only");
    constexpr int NT = kL2Threads;
    constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + kL2NQ;          // named barrier ids
    extern __shared__ __align__(16) uint8_t l2_smem[];
    uint32_t *Q = reinterpret_cast<uint32_t *>(l2_smem);
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

    // zero rows (row index 0 = no source selected) of every buffer
    for (int t = tid; t < kL2NQ * kL2QS; t += NT) Q[(t / kL2QS) * kL2QWords + t % kL2QS] = 0u;
    __syncthreads();

    if (warp >= kL2GW) {
        // ======================= builders
        const int bt = tid - 32 * kL2GW;                       // 0 .. 127
        uint32_t aj = 0, aw0 = 0;                              // source cursor
        int ast = 0;
        size_t ag = tile_g(0, aw0);
        uint32_t ar[kL2NQ][kL2BWords][SG];
        auto load = [&](uint32_t (&a)[kL2BWords][SG]) {      // the cursor's step, then advance
            const bool live = aj < ntj;
            const uint8_t *Ag = p.A + ag * (size_t)p.N * p.M;
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = ast * SG + j;
                const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
#pragma unroll
                for (int u = 0; u < kL2BWords; u++) {
                    const uint32_t wd = aw0 + (uint32_t)bt + 32u * kL2BW * u;
                    a[u][j] = (live && i < p.N && wd < p.Mw) ? __ldg(row + wd) : 0u;
                }
            }
            if (++ast == p.NS) {
                ast = 0;
                aj++;
                ag = tile_g(aj, aw0);
            }
        };
        uint32_t cj = 0, cw0 = 0;                              // coefficient cursor (first builder warp)
        int cst = 0;
        size_t cg = tile_g(0, cw0);
        // raw coefficient bytes of lane k for the cursor's step (first builder warp;
        // prefetched three steps ahead like the source words), then advance
        auto load_c = [&](uint32_t (&c)[SG]) {
            const uint8_t *Cg = p.C + cg * (size_t)p.N * p.K;
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = cst * SG + j;
                c[j] = (cj < ntj && i < p.N && lane < p.K) ? (uint32_t)__ldg(Cg + (size_t)i * p.K + lane) : 0u;
            }
            if (++cst == p.NS) {
                cst = 0;
                cj++;
                cg = tile_g(cj, cw0);
            }
        };
        uint32_t cr[kL2NQ][SG];
        auto bstep = [&](uint32_t s, int b, uint32_t (&a)[kL2BWords][SG], uint32_t (&c)[SG]) {
            if (s >= kL2NQ) nbar_sync(BAR_EMPTY + b, NT);       // gatherers done with step s-NQ
            uint32_t *q = Q + b * kL2QWords;
#pragma unroll
            for (int u = 0; u < kL2BWords; u++) build_word<F, kL2QS>(q + bt + 32 * kL2BW * u, a[u]);
            if (warp == kL2GW) {
                uint8_t cb[SG];
#pragma unroll
                for (int j = 0; j < SG; j++) cb[j] = (uint8_t)c[j];
                idx[b * 32 + lane] = (uint8_t)L::index(cb);
            }
            nbar_arrive(BAR_FULL + b, NT);
            load(a);                                           // step s + 3
            if (warp == kL2GW) load_c(c);
        };
        load(ar[0]);
        load(ar[1]);
        load(ar[2]);
        if (warp == kL2GW) {
            load_c(cr[0]);
            load_c(cr[1]);
            load_c(cr[2]);
        }
#pragma unroll 1
        for (uint32_t s = 0; s < total; s += 3) {
            bstep(s, 0, ar[0], cr[0]);
            if (s + 1 < total) bstep(s + 1, 1, ar[1], cr[1]);
            if (s + 2 < total) bstep(s + 2, 2, ar[2], cr[2]);
        }
        // consume the gatherers' last NQ EMPTY signals
        for (uint32_t s = max(total, (uint32_t)kL2NQ); s < total + kL2NQ; s++) nbar_sync(BAR_EMPTY + s % kL2NQ, NT);
        return;
    }

    // ======================= gatherers: lane = coded packet k, words 32 warp .. 32 warp + 31
    uint32_t *myscr = scr + warp * 32 * kL2ScrS;
    uint32_t acc[32];
#pragma unroll
    for (int w = 0; w < 32; w++) acc[w] = 0u;
    int st_g = 0;
    uint32_t j_g = 0;
    auto gstep = [&](uint32_t s, int b) {
        nbar_sync(BAR_FULL + b, NT);
        const uint32_t r = idx[b * 32 + lane];
        const uint32_t *row = Q + b * kL2QWords + r * kL2QS + warp * 32;
#pragma unroll
        for (int w = 0; w < 32; w++) acc[w] ^= row[w];
        nbar_arrive(BAR_EMPTY + b, NT);
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
