// encode_lanek.cuh -- batched RLNC encode with the coded-packet index k on the
// lanes ("lane = k" layout), shared-memory product tables and warp
// specialisation.  All four fields.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Why: in the column layout (encode_kernels.cuh) every (i, k, word) costs ALU
// instructions (>= 4 for GF(256)) and the kernel is ALU-bound.  Here the
// multiply becomes a shared-memory gather that the LSU pipe serves:
//   * a "step" consumes SG source packets (SG = 4 for GF(2), 2 for GF(4), 1
//     otherwise).  For every word w of the CTA's tile, builder warps write the
//     16 XOR-combinations of four generator values P0..P3 of the step:
//        Q[r][w] = XOR_{j : bit j of r} P_j[w]            r < 16
//       GF(2):   P_j = a_{4s+j}                  (r = the 4 coefficient bits)
//       GF(4):   P = a_{2s}, x a_{2s}, a_{2s+1}, x a_{2s+1}   (r = c0 | c1 << 2)
//       GF(16):  P_j = x^j a_s                   (r = c: Q[c] = c * a)
//       GF(256): as GF(16) for the low nibble of c, plus 16 more rows built
//                from x^4 a .. x^7 a for the high nibble
//     i.e. the paper's split-table idea (Alg. 1) with the
//     roles of data and coefficient exchanged (a "four Russians" table over
//     the coefficient bits), built from the xtime chain by linearity over GF(2);
//   * gatherer warps: lane = coded packet k (32 per warp), each lane reads the
//     row r of ITS coefficients, so one warp-wide LDS gathers 32 products of
//     the same source word (<= 16 distinct rows; odd row stride puts them in
//     distinct banks: one wavefront); WT words per lane accumulate in
//     registers;
//   * Q is triple-buffered between builders and gatherers (named barriers
//     FULL / EMPTY); builders load the source words of a step straight into
//     registers three steps ahead (no shared-memory staging: the smem pipe is
//     the binding resource, so staging would cost ~11% of its wavefronts).
// Per (step, k, word): 1 LDS + 1 LOP3 (GF(256): 2 LDS + 1 LOP3); the table
// build (15 or 30 words per source word) is shared by the CTA's 32*KG lanes.
//
// Geometry (LkGeom): KG = 2 k-groups (64 coded packets per CTA, 48 words per
// lane, 384-word tiles, one CTA per SM) for K > 32; KG = 1 (32 coded packets,
// 32 words per lane, 256-word tiles, three CTAs per SM so that one CTA's
// prologue / epilogue overlaps the others' streaming) otherwise.
#pragma once
#include <cstdint>

#include "encode_kernels.cuh"   // cp_async4
#include "gf_device.cuh"

namespace gfr {

constexpr int kLkWG = 8;                  // word groups (gatherer warps per k-group)
constexpr int kLkBuildWarps = 4;
constexpr int kLkSteps = 4;               // cp.async ring depth in steps
constexpr int kLkNQ = 3;                  // Q buffers between builders and gatherers

// WIDE (GF(2) with KG = 1): 64 words per gatherer lane, two CTAs per SM
// (C5 GF(2): 1649 vs 1610 GB/s with 32 words and three CTAs; GF(4) is the
// other way round: 1047 vs 1093)
template <int KG, bool WIDE = false> struct LkGeom {
    static constexpr int WT = KG == 1 ? (WIDE ? 64 : 32) : 48;   // words per gatherer lane
    static constexpr int WG = KG == 4 ? 4 : kLkWG;        // word groups
    static constexpr int TW = WT * WG;                    // words per tile
    // V2 (KG = 1: C5): 64-bit gathers. Q row stride even with QS / 2 odd, so
    // that rows are 8-byte aligned and the 16 possible rows of a half-warp's
    // LDS.64 sit in 16 distinct 8-byte bank slots (half the LSU instructions of
    // LDS.32 for the same wavefronts; ncu: the LSU instruction pipe was 74% busy
    // against 68% for the wavefronts).  C5 GF(2) +1.1%, GF(4) +3.3%; with
    // KG = 2 it measured 3% slower, so KG > 1 keeps 32-bit gathers, odd stride.
    static constexpr bool V2 = KG == 1;
    static constexpr int QS = V2 ? TW + 2 : TW + 1;
    static_assert(V2 ? (QS / 2) % 2 == 1 : QS % 2 == 1, "Q row stride");
    static constexpr int BWORDS = (TW + 32 * kLkBuildWarps - 1) / (32 * kLkBuildWarps);
    static constexpr int THREADS = 32 * (KG * WG + kLkBuildWarps);
    static constexpr int MINB = KG == 1 ? (WIDE ? 2 : 3) : 1;   // CTAs per SM targeted
};

struct LanekParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    size_t M;          // bytes per packet
    uint32_t Mw;       // words per packet
    size_t batch;
    int N, K;
    int qmask;
    int tiles;         // word tiles per packet
    int k_tiles;       // ceil(K / (32 KG))
    // fused Freivalds check (VT > 0 instantiations, KG <= 2: a CTA's coded
    // packets are exactly one block of 64, or all K <= 32; gf_encode_verify_batch)
    const uint8_t *U;      // [batch][kblocks][2][N]: u_jbi = sum_{k in block b} r_jk C[i][k]
    const uint32_t *RB;    // [batch][2][kw]: bit k of word k / 32 = r_jk
    int kw;
    unsigned long long *mismatch;
    uint64_t fault;        // harness fault injection (FT): g << 32 | k << 20 | word
};

template <int F> struct LkField;
template <> struct LkField<2> {
    static constexpr int kRows = 16, kSG = 4;
    __device__ __forceinline__ static uint32_t index(const uint8_t *c) {
        return (c[0] & 1u) | (c[1] & 1u) << 1 | (c[2] & 1u) << 2 | (c[3] & 1u) << 3;
    }
};
template <> struct LkField<4> {
    static constexpr int kRows = 16, kSG = 2;
    __device__ __forceinline__ static uint32_t index(const uint8_t *c) { return (c[0] & 3u) | (c[1] & 3u) << 2; }
};
template <> struct LkField<16> {
    static constexpr int kRows = 16, kSG = 1;
    __device__ __forceinline__ static uint32_t xtime(uint32_t a)
    {
        return ((a << 1) & 0xEEEEEEEEu) ^ (((a >> 3) & 0x11111111u) * 3u);
    }
    __device__ __forceinline__ static uint32_t index(const uint8_t *c) { return c[0] & 15u; }
};
template <> struct LkField<256> {
    static constexpr int kRows = 32, kSG = 1;
    __device__ __forceinline__ static uint32_t xtime(uint32_t a)
    {
        return ((a << 1) & 0xFEFEFEFEu) ^ (((a >> 7) & 0x01010101u) * 0x1Bu);
    }
    __device__ __forceinline__ static uint32_t index(const uint8_t *c) { return c[0]; }
};

__device__ __forceinline__ void nbar_sync(int id, int n)
{
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n)
{
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory");
}

// rows 1..15 of Q for one word: XOR combinations of p0..p3 (11 XORs)
template <int QS>
__device__ __forceinline__ void store_nibble_products(uint32_t *q, uint32_t p0, uint32_t p1, uint32_t p2,
                                                      uint32_t p3)
{
    const uint32_t q3 = p0 ^ p1, q5 = p2 ^ p0, q6 = p2 ^ p1, q7 = q6 ^ p0;
    q[1 * QS] = p0;  q[2 * QS] = p1;  q[3 * QS] = q3;  q[4 * QS] = p2;
    q[5 * QS] = q5;  q[6 * QS] = q6;  q[7 * QS] = q7;  q[8 * QS] = p3;
    q[9 * QS] = p3 ^ p0;  q[10 * QS] = p3 ^ p1;  q[11 * QS] = p3 ^ q3;
    q[12 * QS] = p3 ^ p2; q[13 * QS] = p3 ^ q5;  q[14 * QS] = p3 ^ q6;
    q[15 * QS] = p3 ^ q7;
}

// generator values of one word for step s (a[j] = word of source packet SG*s+j)
template <int F, int QS>
__device__ __forceinline__ void build_word(uint32_t *q, const uint32_t (&a)[LkField<F>::kSG])
{
    if constexpr (F == 2) {
        store_nibble_products<QS>(q, a[0], a[1], a[2], a[3]);
    } else if constexpr (F == 4) {
        store_nibble_products<QS>(q, a[0], gf4_xtime(a[0]), a[1], gf4_xtime(a[1]));
    } else {
        using L = LkField<F>;
        const uint32_t p1 = L::xtime(a[0]), p2 = L::xtime(p1), p3 = L::xtime(p2);
        store_nibble_products<QS>(q, a[0], p1, p2, p3);
        if constexpr (F == 256) {
            const uint32_t p4 = L::xtime(p3), p5 = L::xtime(p4), p6 = L::xtime(p5), p7 = L::xtime(p6);
            store_nibble_products<QS>(q + 16 * QS, p4, p5, p6, p7);
        }
    }
}

// bits per element; the xtime chain x^b a (b < bits) of a packed word -- u * a
// is the XOR of the chain values selected by the bits of u (the A-side
// projection of the fused check, with u's bits as precomputed masks)
template <int F> __host__ __device__ constexpr int lk_bits() { return F == 2 ? 1 : F == 4 ? 2 : F == 16 ? 4 : 8; }
template <int F>
__device__ __forceinline__ void lk_chain(uint32_t a, uint32_t (&x)[lk_bits<F>()])
{
    x[0] = a;
#pragma unroll
    for (int b = 1; b < lk_bits<F>(); b++) {
        if constexpr (F == 4) x[b] = gf4_xtime(x[b - 1]);
        else if constexpr (F != 2) x[b] = LkField<F>::xtime(x[b - 1]);
    }
}

// VT > 0 (KG <= 2): the fused Freivalds check of gf_encode_verify_batch over
// the CTA's block of coded packets: the builders accumulate y1_j = sum_i u_ji
// a_i for their words from the source words they hold (lk_mul), the
// epilogue accumulates y2_j = sum_k r_jk b_k while it streams the transposed
// tile out of shared memory (one masked XOR per word and projection, shared-
// memory XOR-atomics across warps), and the bytes where y1 != y2 are counted
// into mismatch[g].  FT: the harness fault injection, its own instantiation.
template <int F, int KG, int VT = 0, bool FT = false>
__global__ void __launch_bounds__(LkGeom<KG, F == 2 && KG == 1>::THREADS, LkGeom<KG, F == 2 && KG == 1>::MINB)
encode_lanek_kernel(LanekParams p)
{
    static_assert(VT == 0 || KG <= 2, "fused check: one block of coded packets per CTA");
    using L = LkField<F>;
    using G = LkGeom<KG, F == 2 && KG == 1>;
    constexpr int SG = L::kSG;
    constexpr int WT = G::WT, TW = G::TW, QS = G::QS;
    constexpr int KTL = 32 * KG;                               // coded packets per CTA
    constexpr int GW = KG * G::WG;                             // gatherer warps
    constexpr int NT = G::THREADS;
    constexpr int kQWords = L::kRows * QS;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *Q = smem;                                        // [NQ][rows][QS]
    uint8_t *ccache = reinterpret_cast<uint8_t *>(Q + kLkNQ * kQWords);    // [steps][KTL]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t bid = blockIdx.x;
    const int kt = (int)(bid % (size_t)p.k_tiles);
    const size_t rest = bid / (size_t)p.k_tiles;
    const int tile = (int)(rest % (size_t)p.tiles);
    const size_t g = rest / (size_t)p.tiles;
    const int k0 = kt * KTL;
    const uint32_t w0 = (uint32_t)tile * TW;                   // first word of the tile
    const uint8_t *Ag = p.A + g * (size_t)p.N * p.M;
    const int NS = (p.N + SG - 1) / SG;                        // steps
    // fused check: y1 [VT][TW] (builders), y2 [VT][TW] (XOR-atomics), after the coefficient cache
    uint32_t *y1s = reinterpret_cast<uint32_t *>(ccache + (((size_t)KTL * NS + 15) & ~(size_t)15));
    uint32_t *y2s = y1s + VT * TW;
    (void)y2s;
    // fused check: masks -(bit b of u_ji) per (step, source of the step, projection, b)
    constexpr int WB = lk_bits<F>(), kMaskStep = SG * VT * WB;   // words per step (a multiple of 4)
    static_assert(VT == 0 || kMaskStep % 4 == 0, "mask words per step");
    uint32_t *umask = y2s + VT * TW;
    (void)umask;
    const int kblk = (p.K + 63) / 64, bk = k0 / 64;            // the CTA's block of 64 coded packets
    (void)kblk;
    (void)bk;

    // zero rows (index 0, and 16 for GF(256)) of every buffer; row indices of
    // every (step, k) from the coefficients (rows past N count as c = 0)
    if constexpr (VT > 0) {
        for (int t = threadIdx.x; t < VT * TW; t += blockDim.x) y2s[t] = 0u;
        const uint8_t *Ub = p.U + ((g * (size_t)kblk + (size_t)bk) * 2) * (size_t)p.N;
        for (int e = threadIdx.x; e < NS * kMaskStep; e += blockDim.x) {
            const int b = e % WB, rest = e / WB, j = rest % VT, i = rest / VT;   // i = SG s + source of the step
            const uint32_t u = i < p.N ? __ldg(Ub + (size_t)j * p.N + i) : 0u;
            umask[e] = 0u - ((u >> b) & 1u);
        }
    }
    for (int t = threadIdx.x; t < QS; t += blockDim.x) {
#pragma unroll
        for (int b = 0; b < kLkNQ; b++) {
            Q[b * kQWords + t] = 0u;
            if (F == 256) Q[b * kQWords + 16 * QS + t] = 0u;
        }
    }
    for (int e = threadIdx.x; e < KTL * NS; e += blockDim.x) {
        const int s = e / KTL, kl = e - s * KTL;               // consecutive threads: consecutive k
        uint8_t c[SG];
#pragma unroll
        for (int j = 0; j < SG; j++) {
            const int i = s * SG + j;
            c[j] = (i < p.N && k0 + kl < p.K)
                       ? (uint8_t)(p.C[(g * (size_t)p.N + (size_t)i) * p.K + (size_t)(k0 + kl)] & p.qmask)
                       : (uint8_t)0;
        }
        ccache[e] = (uint8_t)L::index(c);
    }
    __syncthreads();

    constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + kLkNQ, BAR_EPI = 1 + 2 * kLkNQ;   // named barrier ids
    constexpr int BAR_Y1 = 2 + 2 * kLkNQ;                      // fused check: builders' y1 written

    if (warp >= GW) {
        // ---------------- builders: source words straight into registers three
        // steps ahead (no shared-memory staging), write Q[s % NQ]
        const int bt = threadIdx.x - 32 * GW;                  // 0 .. 127
        constexpr int D = kLkNQ;                               // prefetch distance (= NQ: one unrolled round)
        uint32_t ar[D][G::BWORDS][SG];
        uint32_t y1[VT > 0 ? VT : 1][G::BWORDS];
#pragma unroll
        for (int j = 0; j < (VT > 0 ? VT : 1); j++)
#pragma unroll
            for (int u = 0; u < G::BWORDS; u++) y1[j][u] = 0u;

        auto load = [&](int s, uint32_t (&a)[G::BWORDS][SG]) {
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = s * SG + j;
                const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
#pragma unroll
                for (int u = 0; u < G::BWORDS; u++) {
                    const uint32_t tw = (uint32_t)bt + 128u * u;
                    const uint32_t wd = w0 + tw;
                    a[u][j] = (s < NS && i < p.N && tw < (uint32_t)TW && wd < p.Mw) ? __ldg(row + wd) : 0u;
                }
            }
        };
        auto bstep = [&](int s, int b, uint32_t (&a)[G::BWORDS][SG]) {
            if (s >= NS) return;
            if (s >= kLkNQ) nbar_sync(BAR_EMPTY + b, NT);       // gatherers done with step s-NQ
            uint32_t *q = Q + b * kQWords;
#pragma unroll
            for (int u = 0; u < G::BWORDS; u++) {
                const int tw = bt + 128 * u;
                if (tw < TW) build_word<F, QS>(q + tw, a[u]);
            }
            nbar_arrive(BAR_FULL + b, NT);
            if constexpr (VT > 0) {                            // y1_j += u_ji a_i (before the loads reuse a)
                uint32_t m[kMaskStep];                          // this step's masks (broadcast loads)
#pragma unroll
                for (int c = 0; c < kMaskStep; c += 4) {
                    const uint4 mv = *reinterpret_cast<const uint4 *>(umask + s * kMaskStep + c);
                    m[c] = mv.x; m[c + 1] = mv.y; m[c + 2] = mv.z; m[c + 3] = mv.w;
                }
#pragma unroll
                for (int jj = 0; jj < SG; jj++)
#pragma unroll
                    for (int v = 0; v < G::BWORDS; v++) {
                        uint32_t x[WB];                             // x^b a, shared by the projections
                        lk_chain<F>(a[v][jj], x);
#pragma unroll
                        for (int j = 0; j < VT; j++)
#pragma unroll
                            for (int b = 0; b < WB; b++) y1[j][v] ^= x[b] & m[(jj * VT + j) * WB + b];
                    }
            }
            load(s + D, a);
        };
#pragma unroll
        for (int d = 0; d < D; d++) load(d, ar[d]);
#pragma unroll 1
        for (int s = 0; s < NS; s += D) {
            bstep(s, 0, ar[0]);
            bstep(s + 1, 1, ar[1]);
            bstep(s + 2, 2, ar[2]);
        }
        static_assert(D == 3, "builder loop unrolled for three Q buffers");
        if constexpr (VT > 0) {
#pragma unroll
            for (int v = 0; v < G::BWORDS; v++) {
                const int tw = bt + 128 * v;
                if (tw < TW)
#pragma unroll
                    for (int j = 0; j < VT; j++) y1s[j * TW + tw] = y1[j][v];
            }
            nbar_arrive(BAR_Y1, NT);
        }
        // consume the gatherers' last NQ EMPTY signals
        for (int s = max(NS, kLkNQ); s < NS + kLkNQ; s++) nbar_sync(BAR_EMPTY + s % kLkNQ, NT);
        return;
    }

    // ---------------- gatherers: lane = coded packet k, WT words per lane
    const int kl = (warp % KG) * 32 + lane;                    // local k
    const int wg = warp / KG;                                  // word group
    const uint8_t *ccol = ccache + kl;                         // row index of step s at ccol[KTL s]
    uint32_t acc[WT];
#pragma unroll
    for (int w = 0; w < WT; w++) acc[w] = 0u;

#pragma unroll 1
    for (int s = 0; s < NS; s++) {
        const uint32_t r = ccol[s * KTL];
        const int b = s % kLkNQ;
        nbar_sync(BAR_FULL + b, NT);
        const uint32_t *q = Q + b * kQWords + wg * WT;
        if constexpr (!G::V2) {
            const uint32_t *lo = q + (F == 256 ? (r & 15u) : r) * QS;
            const uint32_t *hi = q + (16u + (r >> 4)) * QS;
#pragma unroll
            for (int w = 0; w < WT; w++) acc[w] ^= F == 256 ? lo[w] ^ hi[w] : lo[w];
        } else if (F == 256) {
            const uint2 *lo = reinterpret_cast<const uint2 *>(q + (r & 15u) * QS);
            const uint2 *hi = reinterpret_cast<const uint2 *>(q + (16u + (r >> 4)) * QS);
#pragma unroll
            for (int v = 0; v < WT / 2; v++) {
                const uint2 x = lo[v], y = hi[v];
                acc[2 * v] ^= x.x ^ y.x;
                acc[2 * v + 1] ^= x.y ^ y.y;
            }
        } else {
            const uint2 *lo = reinterpret_cast<const uint2 *>(q + r * QS);
#pragma unroll
            for (int v = 0; v < WT / 2; v++) {
                const uint2 x = lo[v];
                acc[2 * v] ^= x.x;
                acc[2 * v + 1] ^= x.y;
            }
        }
        nbar_arrive(BAR_EMPTY + b, NT);
    }

    if constexpr (FT) {                                        // harness: one wrong byte
        if (g == ((p.fault >> 32) & 0x7FFFFFFFu) && k0 + kl == (int)((p.fault >> 20) & 0xFFFu)) {
            const uint32_t fw = (uint32_t)p.fault & 0xFFFFFu;
#pragma unroll
            for (int w = 0; w < WT; w++)
                if (w0 + (uint32_t)(wg * WT + w) == fw) acc[w] ^= 0x5Au;
        }
    }
    // ---- epilogue: transpose through shared memory so that each warp writes
    // contiguous runs of one coded packet (the Q buffers are free once every
    // gatherer passed its last step: named barrier over the gatherers only)
    constexpr int OS = G::V2 ? TW + 2 : TW + 1;                 // V2: even, OS / 2 odd (64-bit stores conflict-free)
    // rows of coded packets staged per pass: the largest of KTL, KTL/2, ... (>= 32)
    // that fits in the Q buffers
    constexpr int kFit = (kLkNQ * kQWords) / OS;
    constexpr int kRowsPerPass = KTL <= kFit ? KTL : (KTL / 2 <= kFit ? KTL / 2 : (KTL / 4 <= kFit ? KTL / 4 : 32));
    constexpr int kPasses = KTL / kRowsPerPass;
    static_assert(kRowsPerPass * kPasses == KTL && kRowsPerPass % 32 == 0, "epilogue passes");
    uint32_t *ot = Q;                                           // [rows per pass][OS]
    uint32_t y2p[VT > 0 ? VT : 1][TW / 32];                     // fused check: this thread's words' partial y2
#pragma unroll
    for (int j = 0; j < (VT > 0 ? VT : 1); j++)
#pragma unroll
        for (int n = 0; n < TW / 32; n++) y2p[j][n] = 0u;
    (void)y2p;
    const uint32_t nw = min((uint32_t)TW, p.Mw - w0);
#pragma unroll 1
    for (int h = 0; h < kPasses; h++) {
        nbar_sync(BAR_EPI, 32 * GW);
        if (kl / kRowsPerPass == h) {
            const int r = kl - h * kRowsPerPass;
            if constexpr (G::V2) {
                uint2 *o2 = reinterpret_cast<uint2 *>(ot + r * OS + wg * WT);
#pragma unroll
                for (int v = 0; v < WT / 2; v++) o2[v] = make_uint2(acc[2 * v], acc[2 * v + 1]);
            } else {
#pragma unroll
                for (int w = 0; w < WT; w++) ot[r * OS + wg * WT + w] = acc[w];
            }
        }
        nbar_sync(BAR_EPI, 32 * GW);
        const int kbase = k0 + h * kRowsPerPass;
        for (int r = warp; r < kRowsPerPass; r += GW) {
            if (kbase + r >= p.K) break;
            uint32_t *row = reinterpret_cast<uint32_t *>(p.B + (g * (size_t)p.K + (size_t)(kbase + r)) * p.M) + w0;
            if constexpr (VT > 0) {
                const int k = kbase + r;
                uint32_t m[VT];
#pragma unroll
                for (int j = 0; j < VT; j++) m[j] = 0u - ((__ldg(p.RB + (g * 2 + j) * (size_t)p.kw + (k >> 5)) >> (k & 31)) & 1u);
#pragma unroll
                for (int n = 0; n < TW / 32; n++) {
                    const uint32_t w = (uint32_t)(lane + 32 * n);
                    if (w < nw) {
                        const uint32_t x = ot[r * OS + w];
                        row[w] = x;
#pragma unroll
                        for (int j = 0; j < VT; j++) y2p[j][n] ^= x & m[j];
                    }
                }
            } else {
                for (uint32_t w = lane; w < nw; w += 32) row[w] = ot[r * OS + w];
            }
        }
    }
    if constexpr (VT > 0) {
        // combine the warps' partial y2 (shared-memory XOR-atomics), wait for the
        // builders' y1, count the differing bytes
#pragma unroll
        for (int n = 0; n < TW / 32; n++)
#pragma unroll
            for (int j = 0; j < VT; j++)
                if (y2p[j][n]) atomicXor(y2s + j * TW + lane + 32 * n, y2p[j][n]);
        nbar_sync(BAR_Y1, NT);
        uint32_t bad = 0;
        for (int w = threadIdx.x; w < (int)nw; w += 32 * GW)
#pragma unroll
            for (int j = 0; j < VT; j++) bad += nz_bytes(y1s[j * TW + w] ^ y2s[j * TW + w]);
        bad = __reduce_add_sync(0xffffffffu, bad);
        if (lane == 0 && bad) atomicAdd(p.mismatch + g, (unsigned long long)bad);
    }
}

template <int F, int KG, int VT = 0>
__host__ __device__ constexpr size_t lk_smem_bytes(int N)
{
    using G = LkGeom<KG, F == 2 && KG == 1>;
    return (size_t)kLkNQ * LkField<F>::kRows * G::QS * 4 +
           (((size_t)32 * KG * ((N + LkField<F>::kSG - 1) / LkField<F>::kSG) + 15) & ~(size_t)15) +
           (size_t)2 * VT * G::TW * 4 +
           (size_t)VT * ((N + LkField<F>::kSG - 1) / LkField<F>::kSG) * LkField<F>::kSG * lk_bits<F>() * 4;
}

}  // namespace gfr
