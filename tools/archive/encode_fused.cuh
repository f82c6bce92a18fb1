// encode_fused.cuh -- batched RLNC encode (Eq. 2) with the
// CTA's word tile split between two pipes:
//
//   words [0, TWL)   lane-k path (encode_lanek.cuh): builders write 16-row
//                    combination tables per step, gatherer warps (lane = coded
//                    packet k) gather them -> shared-memory pipe;
//   words [TWL, TW)  column path (encode_kernels.cuh engines): lane = word,
//                    coefficients warp-uniform, PRMT / LOP3 / IMAD per
//                    (i, k, word) -> ALU and FMA pipes.
//
// The lane-k kernel alone leaves the ALU pipe ~2/3 idle and the column kernel
// alone leaves the shared-memory pipe idle; splitting each tile lets both
// pipes work on the same source stream.  Both paths
// read the same cp.async ring filled by the builder warps; the FULL / EMPTY
// named barriers that hand the Q tables to the gatherers also hand the ring
// slots to the column warps.  The ring has NQ - 1 extra slots so that a slot
// is never refilled while a column warp that is up to NQ steps behind may
// still read it.
#pragma once
#include <cstdint>

#include "encode_kernels.cuh"
#include "encode_lanek.cuh"

namespace gfr {

constexpr int kFuWT = 32;                 // words per gatherer lane
constexpr int kFuKTC = 16;                // coded packets per column warp
constexpr int kFuWC = 2;                  // words per column lane
constexpr int kFuSpan = 32 * kFuWC;       // words per column warp (64)
constexpr int kFuRing = kLkSteps + kLkNQ - 1;   // ring slots (steps)

template <int KG, int WGL, int CWS> struct FuGeom {
    static constexpr int KTL = 32 * KG;                   // coded packets per CTA
    static constexpr int TWL = WGL * kFuWT;               // lane-k words
    static constexpr int TWC = CWS * kFuSpan;             // column words
    static constexpr int TW = TWL + TWC;
    static constexpr int QS = TWL + 1;                    // odd
    static constexpr int GW = KG * WGL;                   // gatherer warps
    static constexpr int CW = (KTL / kFuKTC) * CWS;       // column warps
    static constexpr int BWARPS = kLkBuildWarps;
    static constexpr int THREADS = 32 * (GW + CW + BWARPS);
    static constexpr int MINB = THREADS <= 512 ? 2 : 1;
    static constexpr int NI = 16;                         // column table chunk (sources)
};

template <int F, int KG, int WGL, int CWS>
__global__ void __launch_bounds__(FuGeom<KG, WGL, CWS>::THREADS, FuGeom<KG, WGL, CWS>::MINB)
encode_fused_kernel(LanekParams p, const uint32_t *__restrict__ tabs)
{
    using L = LkField<F>;
    using G = FuGeom<KG, WGL, CWS>;
    using E = Engine<F, kFuKTC>;
    constexpr int SG = L::kSG;
    constexpr int KTL = G::KTL, TWL = G::TWL, TW = G::TW, QS = G::QS;
    constexpr int GW = G::GW, CW = G::CW, NT = G::THREADS, NI = G::NI;
    constexpr int kQWords = L::kRows * QS;
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *Q = smem;                                                   // [NQ][rows][QS]
    uint32_t *ring = Q + kLkNQ * kQWords;                                 // [kFuRing][SG][TW]
    uint32_t *ctab = ring + kFuRing * SG * TW;                            // [NI][KTL][EW]
    uint8_t *ccache = reinterpret_cast<uint8_t *>(ctab + NI * KTL * E::EW);   // [steps][KTL]
    const int NS = (p.N + SG - 1) / SG;
    uint8_t *craw = ccache + ((NS * KTL + 15) & ~15);                     // [N][KTL]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t bid = blockIdx.x;
    const int kt = (int)(bid % (size_t)p.k_tiles);
    const size_t rest = bid / (size_t)p.k_tiles;
    const int tile = (int)(rest % (size_t)p.tiles);
    const size_t g = rest / (size_t)p.tiles;
    const int k0 = kt * KTL;
    const uint32_t w0 = (uint32_t)tile * TW;
    const uint8_t *Ag = p.A + g * (size_t)p.N * p.M;

    for (int t = threadIdx.x; t < QS; t += blockDim.x) {
#pragma unroll
        for (int b = 0; b < kLkNQ; b++) {
            Q[b * kQWords + t] = 0u;
            if (F == 256) Q[b * kQWords + 16 * QS + t] = 0u;
        }
    }
    for (int e = threadIdx.x; e < KTL * p.N; e += blockDim.x) {
        const int i = e / KTL, kl = e - i * KTL;
        craw[e] = (k0 + kl < p.K) ? (uint8_t)(p.C[(g * (size_t)p.N + (size_t)i) * p.K + (size_t)(k0 + kl)] & p.qmask)
                                  : (uint8_t)0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < KTL * NS; e += blockDim.x) {
        const int s = e / KTL, kl = e - s * KTL;
        uint8_t c[SG];
#pragma unroll
        for (int j = 0; j < SG; j++) c[j] = s * SG + j < p.N ? craw[(s * SG + j) * KTL + kl] : (uint8_t)0;
        ccache[e] = (uint8_t)L::index(c);
    }
    __syncthreads();

    constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + kLkNQ, BAR_EPI = 1 + 2 * kLkNQ, BAR_COL = 2 + 2 * kLkNQ;

    if (warp >= GW + CW) {
        // ---------------- builders: ring for the whole tile, Q for the lane-k words
        const int bt = threadIdx.x - 32 * (GW + CW);          // 0 .. 127
        const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
        constexpr int BW = (TW + 127) / 128;
        auto issue = [&](int s) {
            if (s < NS) {
#pragma unroll
                for (int j = 0; j < SG; j++) {
                    const int i = s * SG + j;
                    const uint32_t *row = reinterpret_cast<const uint32_t *>(Ag + (size_t)min(i, p.N - 1) * p.M);
                    const uint32_t slot = (uint32_t)((s % kFuRing) * SG + j) * TW;
#pragma unroll
                    for (int u = 0; u < BW; u++) {
                        const uint32_t tw = (uint32_t)bt + 128u * u;
                        if (tw < (uint32_t)TW) {
                            const uint32_t wd = w0 + tw;
                            const bool v = i < p.N && wd < p.Mw;
                            cp_async4(ring_s + (slot + tw) * 4u, v ? row + wd : row, v);
                        }
                    }
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
#pragma unroll 1
        for (int s = 0; s < kLkSteps - 1; s++) issue(s);
#pragma unroll 1
        for (int s = 0; s < NS; s++) {
            const int b = s % kLkNQ;
            if (s >= kLkNQ) nbar_sync(BAR_EMPTY + b, NT);       // everyone done with step s-NQ
            issue(s + kLkSteps - 1);
            asm volatile("cp.async.wait_group %0;" :: "n"(kLkSteps - 1) : "memory");
            uint32_t *q = Q + b * kQWords;
            const uint32_t *slot = ring + (s % kFuRing) * SG * TW;
#pragma unroll
            for (int u = 0; u < (TWL + 127) / 128; u++) {
                const int tw = bt + 128 * u;
                if (tw < TWL) {
                    uint32_t a[SG];
#pragma unroll
                    for (int j = 0; j < SG; j++) a[j] = slot[j * TW + tw];
                    build_word<F, QS>(q + tw, a);
                }
            }
            nbar_arrive(BAR_FULL + b, NT);
        }
        for (int s = max(NS, kLkNQ); s < NS + kLkNQ; s++) nbar_sync(BAR_EMPTY + s % kLkNQ, NT);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        return;
    }

    if (warp >= GW) {
        // ---------------- column warps: words TWL + span*64 + lane + 32 w, 16 coded packets
        const int cw = warp - GW;
        const int kgc = cw % (KTL / kFuKTC);                   // column k-group
        const int span = cw / (KTL / kFuKTC);
        const int kb = kgc * kFuKTC;                           // first local k
        const uint32_t tw0 = (uint32_t)TWL + (uint32_t)span * kFuSpan + (uint32_t)lane;
        uint32_t acc[kFuKTC][kFuWC];
#pragma unroll
        for (int k = 0; k < kFuKTC; k++)
#pragma unroll
            for (int w = 0; w < kFuWC; w++) acc[k][w] = 0u;
        const int ctid = threadIdx.x - 32 * GW;
#pragma unroll 1
        for (int s = 0; s < NS; s++) {
            const int b = s % kLkNQ;
            nbar_sync(BAR_FULL + b, NT);
            const uint32_t *slot = ring + (s % kFuRing) * SG * TW;
#pragma unroll
            for (int j = 0; j < SG; j++) {
                const int i = s * SG + j;
                if (i >= p.N) break;
                if (i % NI == 0) {
                    // resolve coefficients of sources i .. i+NI-1 (column warps only)
                    nbar_sync(BAR_COL, 32 * CW);
                    for (int e = ctid; e < NI * KTL; e += 32 * CW) {
                        const int ie = e / KTL, kk = e - ie * KTL;
                        const uint32_t c = i + ie < p.N ? craw[(i + ie) * KTL + kk] : 0u;
                        E::fill_entry(ctab + (size_t)e * E::EW, tabs + (size_t)c * 16u, kk % kFuKTC);
                    }
                    nbar_sync(BAR_COL, 32 * CW);
                }
                typename E::Word wd[kFuWC];
#pragma unroll
                for (int w = 0; w < kFuWC; w++) wd[w] = E::prep(slot[j * TW + tw0 + 32u * w]);
                E::template apply<kFuWC>(acc, wd, ctab + (size_t)((i % NI) * KTL + kb) * E::EW);
            }
            nbar_arrive(BAR_EMPTY + b, NT);
        }
#pragma unroll
        for (int k = 0; k < kFuKTC; k++) {
            const int kg = k0 + kb + k;
            if (kg < p.K) {
                uint32_t *row = reinterpret_cast<uint32_t *>(p.B + (g * (size_t)p.K + (size_t)kg) * p.M);
#pragma unroll
                for (int w = 0; w < kFuWC; w++) {
                    const uint32_t wd = w0 + tw0 + 32u * w;
                    if (wd < p.Mw) row[wd] = E::kPermuted ? unperm(acc[k][w]) : acc[k][w];
                }
            }
        }
        return;
    }

    // ---------------- gatherers (lane-k words)
    const int kl = (warp % KG) * 32 + lane;
    const int wg = warp / KG;
    const uint8_t *ccol = ccache + kl;
    uint32_t acc[kFuWT];
#pragma unroll
    for (int w = 0; w < kFuWT; w++) acc[w] = 0u;
#pragma unroll 1
    for (int s = 0; s < NS; s++) {
        const uint32_t r = ccol[s * KTL];
        const int b = s % kLkNQ;
        nbar_sync(BAR_FULL + b, NT);
        const uint32_t *q = Q + b * kQWords + wg * kFuWT;
        if (F == 256) {
            const uint32_t *lo = q + (r & 15u) * QS;
            const uint32_t *hi = q + (16u + (r >> 4)) * QS;
#pragma unroll
            for (int w = 0; w < kFuWT; w++) acc[w] ^= lo[w] ^ hi[w];
        } else {
            const uint32_t *lo = q + r * QS;
#pragma unroll
            for (int w = 0; w < kFuWT; w++) acc[w] ^= lo[w];
        }
        nbar_arrive(BAR_EMPTY + b, NT);
    }
    // epilogue through the Q buffers (free: the builders wait for every EMPTY
    // before leaving, and column warps never touch Q)
    constexpr int OS = TWL + 1;
    constexpr int kPasses = (KTL * OS + kLkNQ * kQWords - 1) / (kLkNQ * kQWords);
    constexpr int kRowsPerPass = KTL / kPasses;
    static_assert(kRowsPerPass * kPasses == KTL && kRowsPerPass % 32 == 0, "epilogue passes");
    uint32_t *ot = Q;
    const uint32_t nw = p.Mw > w0 ? min((uint32_t)TWL, p.Mw - w0) : 0u;
#pragma unroll 1
    for (int h = 0; h < kPasses; h++) {
        nbar_sync(BAR_EPI, 32 * GW);
        if (kl / kRowsPerPass == h) {
            const int r = kl - h * kRowsPerPass;
#pragma unroll
            for (int w = 0; w < kFuWT; w++) ot[r * OS + wg * kFuWT + w] = acc[w];
        }
        nbar_sync(BAR_EPI, 32 * GW);
        const int kbase = k0 + h * kRowsPerPass;
        for (int r = warp; r < kRowsPerPass; r += GW) {
            if (kbase + r >= p.K) break;
            uint32_t *row = reinterpret_cast<uint32_t *>(p.B + (g * (size_t)p.K + (size_t)(kbase + r)) * p.M) + w0;
            for (uint32_t w = lane; w < nw; w += 32) row[w] = ot[r * OS + w];
        }
    }
}

template <int F, int KG, int WGL, int CWS>
__host__ __device__ constexpr size_t fu_smem_bytes(int N)
{
    using G = FuGeom<KG, WGL, CWS>;
    constexpr int SG = LkField<F>::kSG;
    const size_t ns = (size_t)(N + SG - 1) / SG;
    return (size_t)kLkNQ * LkField<F>::kRows * G::QS * 4 + (size_t)kFuRing * SG * G::TW * 4 +
           (size_t)G::NI * G::KTL * Engine<F, kFuKTC>::EW * 4 + ((ns * G::KTL + 15) & ~size_t(15)) +
           (size_t)N * G::KTL;
}

}  // namespace gfr
