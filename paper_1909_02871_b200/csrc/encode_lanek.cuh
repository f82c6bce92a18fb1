// encode_lanek.cuh -- batched RLNC encode over GF(16) / GF(256) with the
// coded packet index k on the lanes ("lane = k" layout), shared-memory
// product tables, and warp specialisation.
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// Why: in the column layout (encode_kernels.cuh) every (i, k, word) costs >= 4
// ALU-pipe instructions for GF(256) and the kernel is ALU-bound.  Here the
// multiply becomes a shared-memory lookup that the LSU pipe serves:
//   * for every source packet i and every word w of the CTA's tile, builder
//     warps write the products of a_i[w] with ALL coefficients of a nibble:
//       GF(16):  Q[c][w]     = c * a_i[w],                 c < 16
//       GF(256): Q[c][w]     = c * a_i[w],                 c < 16   (low nibble)
//                Q[16+c][w]  = (c * x^4) * a_i[w],         c < 16   (high nibble)
//     (GF(2)-linearity in c: c*a = c_lo*a + c_hi*(x^4 a)); this is the paper's
//     split-table idea (Alg. 1) with the roles of data and
//     coefficient exchanged, built from the xtime chain a, xa, x^2 a, ...;
//   * gatherer warps: lane = coded packet k (32 per warp), each lane reads
//     the row of ITS coefficient c_ik, so one warp-wide LDS gathers 32
//     different products of the same source word (<= 16 distinct rows; the
//     row stride is odd so the rows sit in distinct banks: one wavefront);
//     acc[w] ^= Q[c_lo][w] ^ Q[16 + c_hi][w], 48 words per lane in registers;
//   * the Q tables are double-buffered: builders fill buffer i&1 while the
//     gatherers read buffer (i-1)&1; named barriers FULL/EMPTY hand them over;
//   * builders also stream the source tile HBM -> smem with a cp.async ring.
// Per (i, k, word): GF(256) 2 LDS + 1 LOP3; GF(16) 1 LDS + 1 LOP3.  The table
// build (15 or 30 products per source word) is amortised over the CTA's 64
// coded packets.
#pragma once
#include <cstdint>

#include "encode_kernels.cuh"   // cp_async4
#include "gf_device.cuh"

namespace gfr {

constexpr int kLkWT = 48;                 // words per gatherer lane
constexpr int kLkWG = 8;                  // word groups per CTA
constexpr int kLkTW = kLkWT * kLkWG;      // words per CTA tile (384)
constexpr int kLkQS = kLkTW + 1;          // Q row stride in words (odd: bank-conflict-free gathers)
constexpr int kLkKT = 64;                 // coded packets per CTA (2 gatherer k-groups)
constexpr int kLkGatherWarps = 16;
constexpr int kLkBuildWarps = 4;
constexpr int kLkThreads = 32 * (kLkGatherWarps + kLkBuildWarps);
constexpr int kLkStages = 4;              // cp.async ring depth (source rows)
constexpr int kLkBuildWords = kLkTW / (32 * kLkBuildWarps);   // words per builder thread (3)

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
    int k_tiles;       // ceil(K / 64)
    int ncpad;         // coefficient cache row length (N rounded up to 4)
};

template <int F> struct LkField;
template <> struct LkField<16> {
    static constexpr int kRows = 16;
    __device__ __forceinline__ static uint32_t xtime(uint32_t a)
    {
        return ((a << 1) & 0xEEEEEEEEu) ^ (((a >> 3) & 0x11111111u) * 3u);
    }
};
template <> struct LkField<256> {
    static constexpr int kRows = 32;
    __device__ __forceinline__ static uint32_t xtime(uint32_t a)
    {
        return ((a << 1) & 0xFEFEFEFEu) ^ (((a >> 7) & 0x01010101u) * 0x1Bu);
    }
};

__device__ __forceinline__ void nbar_sync(int id, int n)
{
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n)
{
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory");
}

// Q rows 1..15 (and 17..31) of one word from its xtime chain
__device__ __forceinline__ void store_nibble_products(uint32_t *q, uint32_t p0, uint32_t p1, uint32_t p2,
                                                      uint32_t p3)
{
    const uint32_t q3 = p0 ^ p1, q5 = p2 ^ p0, q6 = p2 ^ p1, q7 = q6 ^ p0;
    q[1 * kLkQS] = p0;  q[2 * kLkQS] = p1;  q[3 * kLkQS] = q3;  q[4 * kLkQS] = p2;
    q[5 * kLkQS] = q5;  q[6 * kLkQS] = q6;  q[7 * kLkQS] = q7;  q[8 * kLkQS] = p3;
    q[9 * kLkQS] = p3 ^ p0;  q[10 * kLkQS] = p3 ^ p1;  q[11 * kLkQS] = p3 ^ q3;
    q[12 * kLkQS] = p3 ^ p2; q[13 * kLkQS] = p3 ^ q5;  q[14 * kLkQS] = p3 ^ q6;
    q[15 * kLkQS] = p3 ^ q7;
}

template <int F>
__global__ void __launch_bounds__(kLkThreads, 1) encode_lanek_kernel(LanekParams p)
{
    using L = LkField<F>;
    extern __shared__ __align__(16) uint32_t smem[];
    constexpr int kQWords = L::kRows * kLkQS;
    uint32_t *Q = smem;                                        // [2][rows][QS]
    uint32_t *ring = Q + 2 * kQWords;                          // [S][TW]
    uint8_t *ccache = reinterpret_cast<uint8_t *>(ring + kLkStages * kLkTW);   // [N][64]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t bid = blockIdx.x;
    const int kt = (int)(bid % (size_t)p.k_tiles);
    const size_t rest = bid / (size_t)p.k_tiles;
    const int tile = (int)(rest % (size_t)p.tiles);
    const size_t g = rest / (size_t)p.tiles;
    const int k0 = kt * kLkKT;
    const uint32_t w0 = (uint32_t)tile * kLkTW;                // first word of the tile
    const uint8_t *Ag = p.A + g * (size_t)p.N * p.M;

    // zero rows (c_lo = 0, c_hi = 0) of both buffers; coefficient cache
    for (int t = threadIdx.x; t < kLkQS; t += blockDim.x) {
#pragma unroll
        for (int b = 0; b < 2; b++) {
            Q[b * kQWords + t] = 0u;
            if (F == 256) Q[b * kQWords + 16 * kLkQS + t] = 0u;
        }
    }
    for (int e = threadIdx.x; e < kLkKT * p.N; e += blockDim.x) {
        const int i = e / kLkKT, kl = e - i * kLkKT;      // consecutive threads: consecutive k
        uint8_t c = 0;
        if (k0 + kl < p.K)
            c = p.C[(g * (size_t)p.N + (size_t)i) * p.K + (size_t)(k0 + kl)] & (uint8_t)p.qmask;
        ccache[e] = c;
    }
    __syncthreads();

    constexpr int NT = kLkThreads;
    constexpr int BAR_FULL = 1, BAR_EMPTY = 3;   // ids 1,2 and 3,4

    if (warp >= kLkGatherWarps) {
        // ---------------- builders: stream a_i into the ring, write Q[i & 1]
        const int bt = threadIdx.x - 32 * kLkGatherWarps;      // 0 .. 127
        const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
        auto issue = [&](int i) {
            if (i < p.N) {
                const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)i * p.M);
                const uint32_t slot = (uint32_t)(i % kLkStages) * kLkTW;
#pragma unroll
                for (int j = 0; j < kLkBuildWords; j++) {
                    const uint32_t tw = (uint32_t)bt + 128u * j;
                    const uint32_t wd = w0 + tw;
                    const bool v = wd < p.Mw;
                    cp_async4(ring_s + (slot + tw) * 4u, v ? row + wd : row, v);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
#pragma unroll 1
        for (int s = 0; s < kLkStages - 1; s++) issue(s);
#pragma unroll 1
        for (int i = 0; i < p.N; i++) {
            issue(i + kLkStages - 1);
            asm volatile("cp.async.wait_group %0;" :: "n"(kLkStages - 1) : "memory");
            if (i >= 2) nbar_sync(BAR_EMPTY + (i & 1), NT);     // gatherers done with row i-2
            uint32_t *q = Q + (i & 1) * kQWords;
            const uint32_t *slot = ring + (i % kLkStages) * kLkTW;
#pragma unroll
            for (int j = 0; j < kLkBuildWords; j++) {
                const int tw = bt + 128 * j;
                const uint32_t a = slot[tw];
                const uint32_t p1 = L::xtime(a), p2 = L::xtime(p1), p3 = L::xtime(p2);
                store_nibble_products(q + tw, a, p1, p2, p3);
                if (F == 256) {
                    const uint32_t p4 = L::xtime(p3), p5 = L::xtime(p4), p6 = L::xtime(p5), p7 = L::xtime(p6);
                    store_nibble_products(q + 16 * kLkQS + tw, p4, p5, p6, p7);
                }
            }
            nbar_arrive(BAR_FULL + (i & 1), NT);
        }
        // consume the gatherers' last two EMPTY signals
        for (int i = max(p.N, 2); i < p.N + 2; i++) nbar_sync(BAR_EMPTY + (i & 1), NT);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        return;
    }

    // ---------------- gatherers: lane = coded packet k, 48 words per lane
    const int kl = (warp & 1) * 32 + lane;                     // local k (0..63)
    const int wg = warp >> 1;                                  // word group (0..7)
    const uint8_t *ccol = ccache + kl;                        // c of row i at ccol[64 i]
    uint32_t acc[kLkWT];
#pragma unroll
    for (int w = 0; w < kLkWT; w++) acc[w] = 0u;

#pragma unroll 1
    for (int i = 0; i < p.N; i++) {
        const uint32_t c = ccol[i * kLkKT];
        nbar_sync(BAR_FULL + (i & 1), NT);
        const uint32_t *q = Q + (i & 1) * kQWords + wg * kLkWT;
        if (F == 256) {
            const uint32_t *lo = q + (c & 15u) * kLkQS;
            const uint32_t *hi = q + (16u + (c >> 4)) * kLkQS;
#pragma unroll
            for (int w = 0; w < kLkWT; w++) acc[w] ^= lo[w] ^ hi[w];
        } else {
            const uint32_t *lo = q + c * kLkQS;
#pragma unroll
            for (int w = 0; w < kLkWT; w++) acc[w] ^= lo[w];
        }
        nbar_arrive(BAR_EMPTY + (i & 1), NT);
    }

    // ---- epilogue: transpose through shared memory so that each warp writes
    // contiguous runs of one coded packet (the Q buffers are free once every
    // gatherer passed its last row: named barrier over the gatherers only)
    constexpr int kLkOS = kLkTW + 1;
    constexpr int kHalves = (2 * L::kRows * kLkQS >= kLkKT * kLkOS) ? 1 : 2;   // GF(16): 2 passes
    uint32_t *ot = Q;                                           // [64 / kHalves][kLkOS]
    const uint32_t nw = min((uint32_t)kLkTW, p.Mw - w0);
#pragma unroll 1
    for (int h = 0; h < kHalves; h++) {
        nbar_sync(5, 32 * kLkGatherWarps);
        if (kHalves == 1 || (warp & 1) == h) {
            const int r = kHalves == 1 ? kl : lane;
#pragma unroll
            for (int w = 0; w < kLkWT; w++) ot[r * kLkOS + wg * kLkWT + w] = acc[w];
        }
        nbar_sync(5, 32 * kLkGatherWarps);
        const int rows = kLkKT / kHalves, kbase = k0 + h * rows;
        for (int r = warp; r < rows; r += kLkGatherWarps) {
            if (kbase + r >= p.K) break;
            uint32_t *row = reinterpret_cast<uint32_t *>(p.B + (g * (size_t)p.K + (size_t)(kbase + r)) * p.M) + w0;
            for (uint32_t w = lane; w < nw; w += 32) row[w] = ot[r * kLkOS + w];
        }
    }
}

}  // namespace gfr
