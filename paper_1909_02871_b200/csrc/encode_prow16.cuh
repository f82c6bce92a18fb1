// encode_prow16.cuh -- the product-row encode for GF(16) with NIBBLE-indexed
// tables.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// In GF(16) an element is a nibble and the product of two nibbles is a nibble,
// so the product table can be indexed by ONE source element (16 rows, the
// paper's nibble split tables, Alg. 1, turned around as in
// encode_prow.cuh) and still return two coded packets per gathered byte:
//     T[v][s][k] = C[g][s][k] * v            v = 0..15
//     row v, 16-byte chunk (s, h) = T[v][s][32h + 2b] | T[v][s][32h + 2b + 1] << 4, b < 16
// A 16-byte gather for the low (or high) nibble of a source byte returns the
// products of that element with 32 coded packets: one gathered byte per
// byte-madd, as with the byte-indexed tables, but a step's table is 16 rows
// (4 KiB with the duplicated slots below) instead of 256 rows (64 KiB), so the
// table stores that cost the byte-indexed GF(256) kernel 16% of its shared-
// memory traffic on C3 all but vanish.
//
// Row layout (256 B per value v) and conflict freedom.  Slot (16 B) index
//     q = (s & 1) * 4 + h * 2 + n + (s >> 1) * 8
// for source s < 4, coefficient half h (32 coded packets) and nibble half n;
// the two n slots hold the same products (the low- and high-nibble lanes read
// different rows, so they need different bank slots).  The 8 lanes of a
// quarter-warp are (word jw, half h, nibble n); at sub-step t word jw reads
// source (jw + t) & 3, so the two words read sources of opposite parity and
// the 8 slots (q mod 8) are distinct for ANY data: 4 wavefronts per LDS.128.
// Address: prmt(nibble-spread source word, col, sel) = v * 256 + col.
//
// Write-back: the lanes of a pair (n = 0, 1) hold the low- and high-nibble
// products of the same bytes; one shuffle exchanges them, lane n = 0 forms the
// even and lane n = 1 the odd coded packets of each packed byte, then the same
// 4x4 byte transpose as encode_prow.cuh gives whole coded-packet words.
//
// Everything else (persistent CTAs, 4 producer + 12 gatherer warps, BUILT /
// DONE mbarrier rings, three table buffers, source prefetch) is the protocol of
// encode_prow.cuh; 64 coded packets per CTA.
#pragma once
#include <cstdint>

#include "encode_prow.cuh"

namespace gfr {

constexpr uint32_t kNbTab0 = 0x1000u;             // tables u = 0, 1, 2 at kNbTab0 + u * 0x1000
constexpr uint32_t kNbSmemEnd = kNbTab0 + 3 * 0x1000u;

__global__ void __launch_bounds__(kPrThreads, 1) encode_prow16_kernel(ProwParams p)
{
    constexpr int KC = 64, kS = 4, R = 4, GW = 12;
    constexpr uint32_t kBuilt = kPrBar, kDone = kPrBar + 32;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t ntile_cta = p.ntiles > blockIdx.x ? (p.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const uint32_t ntj = (uint32_t)ntile_cta;
    const uint32_t total = ntj * (uint32_t)p.NS;

    auto tile_of = [&](uint32_t j) {
        const size_t t = blockIdx.x + (size_t)(j < ntj ? j : 0u) * gridDim.x;
        PrTile r;
        const int kt = (int)(t % (size_t)p.k_tiles);
        const size_t rest = t / (size_t)p.k_tiles;
        r.w0 = (uint32_t)(rest % (size_t)p.tiles) * kPrTW;
        r.g = rest / (size_t)p.tiles;
        r.k0 = kt * KC;
        return r;
    };

    if (tid == 0) {
#pragma unroll
        for (int b = 0; b < 4; b++) {
            mbar_init(kBuilt + 8 * b, kPrPW);
            mbar_init(kDone + 8 * b, GW);
        }
#pragma unroll
        for (int b = 0; b < 4; b++) mbar_arrive_n(kDone + 8 * b, GW);    // DONE(-4 .. -1)
    }
    __syncthreads();

    if (warp >= GW) {
        // ======================= producers: 16-row nibble tables
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" :: "n"(kPrPRegs));
        const int pt = tid - GW * 32;                           // 0 .. 127
        // thread (v, s, h): the 16-byte chunk of row v for source s, half h,
        // written to both nibble slots n = 0, 1
        const int sh = pt & 7, v = pt >> 3;
        const int s = sh >> 1, h = sh & 1;
        const uint32_t slot0 = (uint32_t)(((s & 1) * 4 + h * 2) + (s >> 1) * 8) * 16u;
        auto build = [&](uint32_t x, uint32_t tab) {
            const uint32_t jt = x / (uint32_t)p.NS, st = x - jt * (uint32_t)p.NS;
            const PrTile T = tile_of(jt);
            const int i = kS * (int)st + s, kb = T.k0 + 32 * h;
            uint32_t cw[8];                                     // 32 coefficient bytes (one element each)
            const uint8_t *cp = p.C + (T.g * (size_t)p.N + (size_t)i) * p.K + kb;
            const bool ok = jt < ntj && i < p.N;
            if (ok && p.cword && kb + 32 <= p.K && (reinterpret_cast<uintptr_t>(cp) & 15u) == 0) {
                const uint4 c0 = __ldg(reinterpret_cast<const uint4 *>(cp));
                const uint4 c1 = __ldg(reinterpret_cast<const uint4 *>(cp) + 1);
                cw[0] = c0.x; cw[1] = c0.y; cw[2] = c0.z; cw[3] = c0.w;
                cw[4] = c1.x; cw[5] = c1.y; cw[6] = c1.z; cw[7] = c1.w;
            } else {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    uint32_t wv = 0u;
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if (ok && kb + 4 * q + e < p.K) wv |= (uint32_t)__ldg(cp + 4 * q + e) << (8 * e);
                    cw[q] = wv;
                }
            }
            // products c * v per byte (element in the low nibble), then two
            // coded packets per byte: b = P[2b] | P[2b + 1] << 4
            uint32_t pw[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                uint32_t c = cw[q] & 0x0F0F0F0Fu, acc = 0u;
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    acc ^= c & (0u - ((uint32_t)(v >> b) & 1u));
                    c = pr_xtime<16>(c);
                }
                pw[q] = acc | (acc >> 4);                       // bytes 0 and 2 hold the packed pairs
            }
            const uint4 out = make_uint4(prmt(pw[0], pw[1], 0x6420u), prmt(pw[2], pw[3], 0x6420u),
                                         prmt(pw[4], pw[5], 0x6420u), prmt(pw[6], pw[7], 0x6420u));
            const uint32_t a = tab + (uint32_t)v * 256u + slot0;
            sts128(a, out);                                     // nibble slot n = 0
            sts128(a + 16u, out);                               // n = 1
        };
        constexpr uint32_t PD = 2;
        auto prefetch_step = [&](uint32_t x) {                  // L2 prefetch of the gatherers' source rows
            const uint32_t j = x / (uint32_t)p.NS, st = x - j * (uint32_t)p.NS;
            if (j >= ntj) return;
            const PrTile T = tile_of(j);
            const uint32_t nw = min((uint32_t)kPrTW, p.Mw - T.w0);
            const uint8_t *row0 = p.A + T.g * (size_t)p.N * p.M + 4 * (size_t)T.w0;
#pragma unroll
            for (int t = 0; t < kS; t++) {
                const int i = kS * (int)st + t;
                if (i >= p.N) break;
                const uintptr_t a = reinterpret_cast<uintptr_t>(row0 + (size_t)i * p.M);
                const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + 4 * (uintptr_t)nw + 15) & ~(uintptr_t)15;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
            }
        };
        if (pt == 0)
            for (uint32_t x = 1; x < PD; x++) prefetch_step(x);
#pragma unroll 1
        for (uint32_t x = 0; x < total; x++) {
            if (pt == 0) prefetch_step(x + PD);
            mbar_wait_sleepy(kDone + ((x - 3) & 3u) * 8u, ((x + 1) >> 2) & 1u);   // DONE(x-3): buffer free
            build(x, kNbTab0 + (x % 3u) * 0x1000u);
            __syncwarp();
            if (lane == 0) mbar_arrive(kBuilt + (x & 3u) * 8u);
        }
        return;
    }

    // ======================= gatherers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" :: "n"(kPrGRegs));
    const int qw = lane >> 3, ql = lane & 7;
    const int jw = ql >> 2, hh = (ql >> 1) & 1, nn = ql & 1;
    constexpr int WQ = 2, WPW = 4 * WQ;
    const uint32_t wbase = (uint32_t)(warp * WPW + qw * WQ + jw);
    constexpr uint32_t kRW = GW * WPW;                          // 96: words per round, R = 4 rounds

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
    uint32_t areg[R][kS];
    size_t soff[kS];
#pragma unroll
    for (int t = 0; t < kS; t++) soff[t] = (size_t)((jw + t) & (kS - 1)) * p.M;
    auto load_a = [&]() {
        const int nsrc = p.N - kS * ast;
#pragma unroll
        for (int t = 0; t < kS; t++) {
            const bool iok = ((jw + t) & (kS - 1)) < nsrc;
            const uint32_t *row = reinterpret_cast<const uint32_t *>(aptr + soff[t]);
#pragma unroll
            for (int r = 0; r < R; r++) areg[r][t] = (iok && (vmask >> r & 1u)) ? __ldg(row + kRW * r) : 0u;
        }
        if (++ast == p.NS) {
            ast = 0;
            aj++;
            seta();
        } else {
            aptr += (size_t)kS * p.M;
        }
    };
    seta();
    uint32_t gmask = vmask;
    load_a();

    uint4 acc[R][4];
#pragma unroll
    for (int r = 0; r < R; r++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);
    int st_g = 0;
    uint32_t j_g = 0;
    // table column of sub-step t: source s = (jw + t) & 3, half hh, nibble slot nn
    uint32_t col[kS];
#pragma unroll
    for (int t = 0; t < kS; t++) {
        const int s = (jw + t) & 3;
        col[t] = (uint32_t)(((s & 1) * 4 + hh * 2 + nn) + (s >> 1) * 8) * 16u;
    }
    const uint32_t nshift = 4u * (uint32_t)nn;

    auto step = [&](uint32_t s, auto U) {
        constexpr uint32_t u = decltype(U)::value;
        mbar_wait(kBuilt + (s & 3u) * 8u, (s >> 2) & 1u);
#pragma unroll
        for (int r = 0; r < R; r++) {
            if (!(gmask >> r & 1u)) continue;
            uint32_t nw[kS];                                   // this lane's nibble of every byte: 0x0v0v0v0v
#pragma unroll
            for (int t = 0; t < kS; t++) nw[t] = (areg[r][t] >> nshift) & 0x0F0F0F0Fu;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const uint32_t sel = 0x5504u | (j << 4);
#pragma unroll
                for (int t = 0; t < kS; t += 2) {
                    const uint4 v0 = lds128_at<kNbTab0 + u * 0x1000u>(prmt(nw[t], col[t], sel));
                    const uint4 v1 = lds128_at<kNbTab0 + u * 0x1000u>(prmt(nw[t + 1], col[t + 1], sel));
                    acc[r][j].x = xor3(acc[r][j].x, v0.x, v1.x);
                    acc[r][j].y = xor3(acc[r][j].y, v0.y, v1.y);
                    acc[r][j].z = xor3(acc[r][j].z, v0.z, v1.z);
                    acc[r][j].w = xor3(acc[r][j].w, v0.w, v1.w);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(kDone + (s & 3u) * 8u);
        load_a();
        if (++st_g == p.NS) {
            st_g = 0;
            // ---- write back: acc[r][j] word c holds, for byte j of word r and
            // coded packets k0 + 32 hh + 8c + 2e + {0, 1} (e < 4: byte e),
            // nibble nn's products in the low / high nibble of each byte
            const PrTile T = tile_of(j_g++);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const uint32_t wd = T.w0 + wbase + kRW * r;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    uint32_t x[4];                              // per byte j: 4 output bytes of this lane's parity
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const uint32_t mine = u4c(acc[r][j], c);
                        const uint32_t other = __shfl_xor_sync(0xffffffffu, mine, 1);
                        const uint32_t L = nn ? other : mine, H = nn ? mine : other;
                        x[j] = nn ? (((L >> 4) & 0x0F0F0F0Fu) | (H & 0xF0F0F0F0u))        // odd coded packets
                                  : ((L & 0x0F0F0F0Fu) | ((H & 0x0F0F0F0Fu) << 4));       // even coded packets
                    }
                    if (wd < p.Mw) {
                        const uint32_t t0 = prmt(x[0], x[1], 0x5140u), t1 = prmt(x[0], x[1], 0x7362u);
                        const uint32_t t2 = prmt(x[2], x[3], 0x5140u), t3 = prmt(x[2], x[3], 0x7362u);
                        const uint32_t y[4] = {prmt(t0, t2, 0x5410u), prmt(t0, t2, 0x7632u),
                                               prmt(t1, t3, 0x5410u), prmt(t1, t3, 0x7632u)};
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const int k = T.k0 + 32 * hh + 8 * c + 2 * e + nn;
                            if (k < p.K)
                                reinterpret_cast<uint32_t *>(p.B + (T.g * (size_t)p.K + (size_t)k) * p.M)[wd] = y[e];
                        }
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; j++) acc[r][j] = make_uint4(0u, 0u, 0u, 0u);
            }
            const PrTile Tn = tile_of(j_g);
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
