// decode_kernels.cuh -- batched decoding support:
// per-generation inversion of the N x N coefficient matrix over F_q by
// Gauss-Jordan elimination, one CTA per generation.
//
// Decoding closes the RLNC loop of Eq. 2: with
// B[k] = sum_i C[i][k] a_i for k < N and D = C^{-1} (C D = I),
//     sum_k D[k][j] B[k] = sum_i a_i sum_k C[i][k] D[k][j] = a_j,
// so decode(B, C) = encode(B, D): the batched encode kernels do the heavy
// part, this kernel only inverts the small matrices.
//
// Row operations work on packed 32-bit words of 4 matrix entries with the
// same byte-permute split tables as the encode kernels (every entry is a
// single field element, so the packed byte product is the element product).
// Columns left of the current pivot are already reduced (zero outside pivot
// rows) and are skipped.
#pragma once
#include <cstdint>

#include "gf_device.cuh"

namespace gfr {

struct InvertParams {
    const uint8_t *C;      // [batch][N][N]
    uint8_t *D;            // [batch][N][N]  inverse (undefined where rank < N)
    int *rank;             // [batch] or nullptr
    const uint32_t *tabs;  // table of tables of the field (16 words per coefficient)
    const uint8_t *inv;    // multiplicative inverses of the field (256 bytes)
    size_t batch;
    int N;
    int qmask;
};

__device__ __forceinline__ PrmtTab tab_of(const uint32_t *stab, uint32_t c)
{
    const uint32_t *t = stab + c * 8u;
    PrmtTab T;
    T.t0lo = t[0]; T.t0hi = t[1]; T.t1lo = t[2]; T.t1hi = t[3]; T.t2 = t[4];
    return T;
}

__device__ __forceinline__ uint32_t mul_word(const PrmtTab &T, uint32_t x)
{
    return unperm(lookup_perm(T, make_sel(x)));
}

// one CTA (256 threads) per generation; dynamic smem: augmented matrix
// [N][RW] words (RW = 2N/4 rounded up) + field tables (256 x 8 words) + inverses
__global__ void __launch_bounds__(256) invert_kernel(InvertParams p)
{
    extern __shared__ __align__(16) uint32_t smem[];
    const int N = p.N;
    const int RW = (2 * N + 3) / 4;                   // words per augmented row
    uint32_t *Mx = smem;                              // [N][RW]
    uint32_t *stab = Mx + (size_t)N * RW;             // [256][8]: T0lo,T0hi,T1lo,T1hi,T2,...
    uint8_t *sinv = reinterpret_cast<uint8_t *>(stab + 256 * 8);
    __shared__ int s_piv;
    __shared__ uint8_t s_fac[256];                    // column entries, read before elimination
    const size_t g = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;

    for (int e = tid; e < 256 * 8; e += nt) {
        const int c = e >> 3, j = e & 7;
        stab[e] = j < 5 ? __ldg(p.tabs + (size_t)c * 16u + j) : 0u;
    }
    for (int e = tid; e < 256; e += nt) sinv[e] = __ldg(p.inv + e);
    uint8_t *Mb = reinterpret_cast<uint8_t *>(Mx);
    const uint8_t *Cg = p.C + g * (size_t)N * N;
    for (int e = tid; e < N * RW * 4; e += nt) {
        const int r = e / (RW * 4), c = e - r * RW * 4;
        uint8_t v = 0;
        if (c < N) v = Cg[(size_t)r * N + c] & (uint8_t)p.qmask;
        else if (c < 2 * N) v = (c - N == r) ? 1 : 0;
        Mb[e] = v;
    }
    __syncthreads();

    // elimination geometry: tpr threads per row (a power of two, tpr * N <= nt)
    int tpr = 1;
    while (tpr * 2 * N <= nt && tpr < 32) tpr *= 2;
    const int rl = tid % tpr, r0 = tid / tpr, rstep = nt / tpr;

    int rank = 0;
    for (int col = 0; col < N; col++) {
        // pivot: first row >= rank with a nonzero entry in this column
        if (tid == 0) s_piv = N;
        __syncthreads();
        for (int r = rank + tid; r < N; r += nt)
            if (Mb[(size_t)r * RW * 4 + col]) atomicMin(&s_piv, r);
        __syncthreads();
        const int piv = s_piv;
        if (piv == N) continue;                       // column without pivot: rank deficient
        const int w0 = col >> 2;                      // words left of w0 are reduced
        // swap pivot row into place and scale it by the inverse of the pivot
        const uint32_t pv = Mb[(size_t)piv * RW * 4 + col];
        const PrmtTab Ts = tab_of(stab, sinv[pv]);
        // every thread has read the pivot before any thread rewrites its word
        // in the swap below (warps > 0 would otherwise race with warp 0)
        __syncthreads();
        for (int w = w0 + tid; w < RW; w += nt) {
            const uint32_t a = Mx[(size_t)piv * RW + w];
            const uint32_t b = Mx[(size_t)rank * RW + w];
            Mx[(size_t)piv * RW + w] = b;
            Mx[(size_t)rank * RW + w] = mul_word(Ts, a);
        }
        __syncthreads();
        for (int r = tid; r < N; r += nt) s_fac[r] = r == rank ? 0 : Mb[(size_t)r * RW * 4 + col];
        __syncthreads();
        // eliminate the column from every other row: TPR threads per row, each
        // loads its row's factor table once per column (no per-element division
        // or table reload)
        for (int r = r0; r < N; r += rstep) {
            const uint32_t f = s_fac[r];
            if (f == 0) continue;
            const PrmtTab T = tab_of(stab, f);
            uint32_t *row = Mx + (size_t)r * RW;
            const uint32_t *prow = Mx + (size_t)rank * RW;
            for (int w = w0 + rl; w < RW; w += tpr) row[w] ^= mul_word(T, prow[w]);
        }
        __syncthreads();
        rank++;
    }
    // D = right half
    uint8_t *Dg = p.D + g * (size_t)N * N;
    for (int e = tid; e < N * N; e += nt) {
        const int r = e / N, c = e - r * N;
        Dg[e] = Mb[(size_t)r * RW * 4 + N + c];
    }
    if (tid == 0 && p.rank) p.rank[g] = rank;
}

// ---- warp-per-matrix inversion for N <= 64 (the C3 decode shape) ----------
// One warp owns one generation's augmented matrix [C | I] (N rows x RW words,
// row stride RW + 1 so that the 32 rows a warp touches per word sit in 32
// banks); no CTA-wide barrier at all -- the CTA version above pays five
// __syncthreads per column.  Per column: pivot by two ballots (lane l holds
// rows l and l + 32), row swap + scaling with one word per lane, then each
// lane eliminates its own rows word by word with the split tables of its
// row's factor (loaded once per column).  The PRMT selectors depend only on
// the pivot row, so lane w computes those of pivot word w once per column
// (from the byte-permuted word, so that the lookups come out in natural byte
// order) and every row update reads them back with one broadcast LDS.128:
// 3 PRMT + 2 LOP3 per row word instead of 12 ALU/FMA operations.  Twelve
// matrices per CTA share the field tables.
constexpr int kInvWarps = 12;            // 12 x 8.4 KB matrices: two CTAs (24 warps) per SM (8: 1.21 ms, 12: 1.16 ms for 16384 64x64 inversions)

__device__ __forceinline__ PrmtTab tab5_of(const uint32_t *stab, uint32_t c)
{
    const uint32_t *t = stab + c * 5u;
    PrmtTab T;
    T.t0lo = t[0]; T.t0hi = t[1]; T.t1lo = t[2]; T.t1hi = t[3]; T.t2 = t[4];
    return T;
}

__global__ void __launch_bounds__(32 * kInvWarps) invert_warp_kernel(InvertParams p)
{
    extern __shared__ __align__(16) uint32_t smem[];
    const int N = p.N;
    const int RW = (2 * N + 3) / 4;                   // words per augmented row
    const int RS = RW + 1;                            // row stride (odd: conflict-free column access)
    uint32_t *stab = smem;                            // [256][5]: T0lo,T0hi,T1lo,T1hi,T2
    uint8_t *sinv = reinterpret_cast<uint8_t *>(stab + 256 * 5);
    uint32_t *ssel_all = stab + 256 * 5 + 64;         // [warps][32 words][4]: pivot-row selectors
    uint32_t *Mall = ssel_all + kInvWarps * 32 * 4;   // [warps][N][RS]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < 256 * 5; e += blockDim.x) {
        const int c = e / 5, j = e - c * 5;
        stab[e] = __ldg(p.tabs + (size_t)c * 16u + j);
    }
    for (int e = tid; e < 256; e += blockDim.x) sinv[e] = __ldg(p.inv + e);
    const size_t g = (size_t)blockIdx.x * kInvWarps + warp;
    const bool live = g < p.batch;
    uint32_t *Mx = Mall + (size_t)warp * N * RS;
    uint32_t *ssel = ssel_all + warp * 32 * 4;
    uint8_t *Mb = reinterpret_cast<uint8_t *>(Mx);
    if (live) {
        const uint8_t *Cg = p.C + g * (size_t)N * N;
        for (int e = lane; e < N * RW * 4; e += 32) {
            const int r = e / (RW * 4), c = e - r * RW * 4;
            uint8_t v = 0;
            if (c < N) v = Cg[(size_t)r * N + c] & (uint8_t)p.qmask;
            else if (c < 2 * N) v = (c - N == r) ? 1 : 0;
            Mb[(size_t)r * RS * 4 + c] = v;
        }
    }
    __syncthreads();                                  // tables ready
    if (!live) return;
    __syncwarp();

    const int ra = lane, rb = lane + 32;              // this lane's rows
    const bool has_a = ra < N, has_b = rb < N;        // has_b is warp-uniform false for N <= 32
    uint32_t *rowa = Mx + (size_t)ra * RS, *rowb = Mx + (size_t)rb * RS;
    int rank = 0;
    for (int col = 0; col < N; col++) {
        const int cw = col >> 2;                      // word of the column
        // pivot: first row >= rank with a nonzero entry in this column
        const bool ha = has_a && ra >= rank && Mb[(size_t)ra * RS * 4 + col] != 0;
        const bool hb = has_b && rb >= rank && Mb[(size_t)rb * RS * 4 + col] != 0;
        const uint32_t ba = __ballot_sync(0xffffffffu, ha), bb = __ballot_sync(0xffffffffu, hb);
        if ((ba | bb) == 0u) continue;                // rank deficient column
        const int piv = ba ? __ffs(ba) - 1 : 32 + __ffs(bb) - 1;
        // swap the pivot row into place and scale it by the pivot's inverse;
        // lane w keeps the selectors of the scaled pivot word w
        const uint32_t pv = Mb[(size_t)piv * RS * 4 + col];
        __syncwarp();
        if (lane >= cw && lane < RW) {
            const uint32_t a = Mx[(size_t)piv * RS + lane], b = Mx[(size_t)rank * RS + lane];
            const uint32_t sa = mul_word(tab5_of(stab, sinv[pv]), a);
            Mx[(size_t)piv * RS + lane] = b;
            Mx[(size_t)rank * RS + lane] = sa;
            const Sel sl = make_sel(prmt(sa, sa, 0x3120u));   // permuted input: natural-order products
            *reinterpret_cast<uint4 *>(ssel + lane * 4) = make_uint4(sl.s0, sl.s1, sl.s2, 0u);
        }
        __syncwarp();
        // eliminate: each lane its rows (factor 0 for the pivot row: no change)
        const uint32_t fa = (has_a && ra != rank) ? Mb[(size_t)ra * RS * 4 + col] : 0u;
        const uint32_t fb = (has_b && rb != rank) ? Mb[(size_t)rb * RS * 4 + col] : 0u;
        __syncwarp();                                 // factors read before any row update
        const PrmtTab Ta = tab5_of(stab, fa), Tb = tab5_of(stab, fb);
        for (int w = cw; w < RW; w++) {
            const uint4 sv = *reinterpret_cast<const uint4 *>(ssel + w * 4);   // broadcast
            const Sel sl{sv.x, sv.y, sv.z};
            if (has_a) rowa[w] ^= lookup_perm(Ta, sl);
            if (has_b) rowb[w] ^= lookup_perm(Tb, sl);
        }
        __syncwarp();
        rank++;
    }
    uint8_t *Dg = p.D + g * (size_t)N * N;
    for (int e = lane; e < N * N; e += 32) {
        const int r = e / N, c = e - r * N;
        Dg[e] = Mb[(size_t)r * RS * 4 + N + c];
    }
    if (lane == 0 && p.rank) p.rank[g] = rank;
}

// ---- GF(2), N <= 64: bit-sliced Gauss-Jordan, one warp per matrix --------
// Over GF(2) an entry is one bit, so a row of [C | I] is 128 bits: lane l
// holds rows l and l + 32 as (C bits, I bits) pairs of 64-bit words.  Per
// column: a ballot over the rows not yet used whose bit is set picks the
// pivot, four shuffles broadcast it, and every other row with the bit set
// XORs it in -- the byte-packed kernels' row operation on 64 entries per
// instruction pair.  No row swaps: the pivot row remembers its column and
// becomes that row of D.
constexpr int kInvG2Warps = 8;

__global__ void __launch_bounds__(32 * kInvG2Warps) invert_gf2_kernel(InvertParams p)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t g = (size_t)blockIdx.x * kInvG2Warps + warp;
    if (g >= p.batch) return;
    const int N = p.N;
    const uint8_t *Cg = p.C + g * (size_t)N * N;
    const bool words = (N % 4) == 0 && (reinterpret_cast<uintptr_t>(p.C) & 3u) == 0;
    auto load_row = [&](int r, uint64_t &c, uint64_t &d) {
        c = 0;
        d = 0;
        if (r >= N) return;
        const uint8_t *row = Cg + (size_t)r * N;
        if (words) {
            for (int q = 0; q < N / 4; q++) {
                const uint32_t x = __ldg(reinterpret_cast<const uint32_t *>(row) + q) & 0x01010101u;
                const uint32_t nib = (x & 1u) | ((x >> 7) & 2u) | ((x >> 14) & 4u) | ((x >> 21) & 8u);
                c |= (uint64_t)nib << (4 * q);
            }
        } else {
            for (int k = 0; k < N; k++) c |= (uint64_t)(__ldg(row + k) & 1u) << k;
        }
        d = 1ull << r;
    };
    uint64_t ca, da, cb, db;
    load_row(lane, ca, da);
    load_row(lane + 32, cb, db);
    int pa = -1, pb = -1;                             // column this row became the pivot of
    int rank = 0;
    for (int col = 0; col < N; col++) {
        const bool sa = (ca >> col) & 1u, sb = (cb >> col) & 1u;
        const uint32_t ba = __ballot_sync(0xffffffffu, sa && pa < 0);
        const uint32_t bb = __ballot_sync(0xffffffffu, sb && pb < 0);
        if ((ba | bb) == 0u) continue;                // no pivot: rank deficient column
        const bool inA = ba != 0u;
        const int pl = inA ? __ffs(ba) - 1 : __ffs(bb) - 1;
        const uint64_t pc = __shfl_sync(0xffffffffu, inA ? ca : cb, pl);
        const uint64_t pd = __shfl_sync(0xffffffffu, inA ? da : db, pl);
        const bool pivA = inA && lane == pl, pivB = !inA && lane == pl;
        if (sa && !pivA) { ca ^= pc; da ^= pd; }
        if (sb && !pivB) { cb ^= pc; db ^= pd; }
        if (pivA) pa = col;
        if (pivB) pb = col;
        rank++;
    }
    // row pcol of D = the I bits of the row that pivoted on pcol, one byte per entry
    uint8_t *Dg = p.D + g * (size_t)N * N;
    const bool dwords = (N % 4) == 0 && (reinterpret_cast<uintptr_t>(p.D) & 3u) == 0;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int pc = h ? pb : pa;
        if (pc < 0) continue;
        const uint64_t d = h ? db : da;
        uint8_t *drow = Dg + (size_t)pc * N;
        if (dwords) {
            for (int q = 0; q < N / 4; q++) {
                const uint32_t nib = (uint32_t)(d >> (4 * q)) & 0xFu;
                reinterpret_cast<uint32_t *>(drow)[q] = (nib * 0x00204081u) & 0x01010101u;   // bit e -> byte e
            }
        } else {
            for (int k = 0; k < N; k++) drow[k] = (uint8_t)((d >> k) & 1u);
        }
    }
    if (lane == 0 && p.rank) p.rank[g] = rank;
}

}  // namespace gfr

namespace gfr {

// ---- on-device Freivalds projections -------------
// U[g][i][j] = sum_k C[g][i][k] * R[g][k][j]  (element products from a q x q
// table).  One thread per (g, i, j).
__global__ void __launch_bounds__(256) project_coeffs_kernel(const uint8_t *C, const uint8_t *R, uint8_t *U,
                                                             const uint8_t *__restrict__ mul, int N, int K,
                                                             int t, size_t batch, int qmask)
{
    const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t per = (size_t)N * t;
    if (e >= per * batch) return;
    const size_t g = e / per;
    const int i = (int)((e % per) / t), j = (int)(e % t);
    const uint8_t *Cg = C + (g * N + i) * (size_t)K;
    const uint8_t *Rg = R + g * (size_t)K * t;
    uint32_t acc = 0;
    for (int k = 0; k < K; k++)
        acc ^= __ldg(mul + (size_t)(Cg[k] & qmask) * 256u + (Rg[(size_t)k * t + j] & qmask));
    U[e] = (uint8_t)acc;
}

// gf_encode_verify_batch (NEXT-4): binary projections r_j (j < t <= 2), applied
// per block of 64 coded packets.  U[g][b][j][i] = sum_{k in block b, r_jk = 1}
// C[g][i][k] (an element of F_q, the A-side coefficient of projection j), and
// RB[g][j][w] = the bits r_jk, k = 32 w .. 32 w + 31.  R: [batch][K][t] bytes,
// r_jk = R[g][k][j] & 1.  One CTA per generation: the bits into shared memory
// (and RB), then one thread per (b, i) reduces the block's coefficient bytes of
// row i four at a time under the byte mask of their four r bits.
__global__ void __launch_bounds__(128) verify_prep_kernel(const uint8_t *C, const uint8_t *R, uint8_t *U,
                                                          uint32_t *RB, int N, int K, int t, int kblocks, int kw,
                                                          size_t batch, int qmask)
{
    extern __shared__ uint32_t srb[];                          // [2][kw]
    const size_t g = blockIdx.x;
    if (g >= batch) return;
    for (int f = threadIdx.x; f < 2 * kw; f += blockDim.x) {
        const int j = f / kw, w = f - j * kw;
        uint32_t bits = 0;
        if (j < t)
            for (int k = 32 * w; k < min(K, 32 * w + 32); k++)
                bits |= (uint32_t)(__ldg(R + (g * K + k) * (size_t)t + j) & 1u) << (k - 32 * w);
        srb[f] = bits;
        RB[g * 2 * (size_t)kw + f] = bits;
    }
    __syncthreads();
    const bool cwd = K % 4 == 0 && (reinterpret_cast<uintptr_t>(C) & 3u) == 0;
    for (int e = threadIdx.x; e < kblocks * N; e += blockDim.x) {
        const int b = e / N, i = e - b * N;
        const uint8_t *Cr = C + (g * N + i) * (size_t)K;
        const int k0 = 64 * b, k1 = min(K, k0 + 64);
        uint32_t acc[2] = {0u, 0u};
        for (int k = k0; k < k1; k += 4) {
            uint32_t word = 0;
            if (cwd && k + 4 <= k1) {
                word = __ldg(reinterpret_cast<const uint32_t *>(Cr + k));
            } else {
                for (int d = 0; d < 4 && k + d < k1; d++) word |= (uint32_t)__ldg(Cr + k + d) << (8 * d);
            }
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const uint32_t nib = (srb[j * kw + (k >> 5)] >> (k & 31)) & 0xFu;   // k % 4 == 0
                // bit d of nib -> 0xFF in byte d (nib * 0x00204081 puts bit d at bit 8 d, no carries)
                acc[j] ^= word & (((nib * 0x00204081u) & 0x01010101u) * 0xFFu);
            }
        }
#pragma unroll
        for (int j = 0; j < 2; j++) {
            uint32_t a = acc[j];
            a ^= a >> 16;
            a ^= a >> 8;
            U[((g * kblocks + b) * 2 + j) * (size_t)N + i] = (uint8_t)(j < t ? (a & (uint32_t)qmask) : 0u);
        }
    }
}

// The same check for the encode kernels without a fused form (plain code,
// after the encode): per (g, byte m), for every block b and projection j,
// y1 = sum_i U[g][b][j][i] * A[g][i][m] and y2 = sum_{k in b, r_jk} B[g][k][m].
// (packed byte products through the split tables: tabs = the field's table of
// tables, 16 words per coefficient)
__global__ void __launch_bounds__(256) verify_plain_kernel(const uint8_t *A, const uint8_t *B, const uint8_t *U,
                                                           const uint32_t *RB, const uint32_t *__restrict__ tabs,
                                                           int N, int K, int kblocks, int kw, size_t M, size_t batch,
                                                           unsigned long long *mismatch)
{
    const size_t g = blockIdx.y;
    const uint8_t *Ag = A + g * (size_t)N * M, *Bg = B + g * (size_t)K * M;
    unsigned long long n = 0;
    for (size_t m = (size_t)blockIdx.x * blockDim.x + threadIdx.x; m < M; m += (size_t)gridDim.x * blockDim.x)
        for (int b = 0; b < kblocks; b++)
            for (int j = 0; j < 2; j++) {
                const uint8_t *Ub = U + ((g * kblocks + b) * 2 + j) * (size_t)N;
                uint32_t y1 = 0, y2 = 0;
                for (int i = 0; i < N; i++) {
                    const uint32_t *t = tabs + (size_t)Ub[i] * 16u;
                    PrmtTab T;
                    T.t0lo = __ldg(t); T.t0hi = __ldg(t + 1); T.t1lo = __ldg(t + 2); T.t1hi = __ldg(t + 3);
                    T.t2 = __ldg(t + 4);
                    y1 ^= mul_word(T, Ag[(size_t)i * M + m]) & 0xFFu;
                }
                for (int k = 64 * b; k < min(K, 64 * b + 64); k++)
                    if ((RB[(g * 2 + j) * kw + (k >> 5)] >> (k & 31)) & 1u) y2 ^= Bg[(size_t)k * M + m];
                n += y1 != y2;
            }
    for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(mismatch + g, n);
}

// The same check, word-parallel and streaming (M % 4 == 0, A and B 4-byte
// aligned): one warp per (generation g, chunk of 128 words), lane = words
// w0 + lane + 32 v (v < 4).  A and B are each read once from HBM; per source i
// and projection j the split tables of u_ji come through warp-uniform loads
// (the field's table of tables stays in L1); y1 accumulates in the permuted
// byte order of lookup_perm and is un-permuted once per block.  r_jk is
// warp-uniform, so y2 is a masked XOR per coded row.  Bytes where y1 != y2 are
// counted per generation (same count as verify_plain_kernel).
constexpr int kVwW = 4;                                       // words per lane
// KB blocks of 64 coded packets per pass over A (C4: K = 256, four blocks in one
// pass): the selectors of a source word are made once for all KB blocks.
template <int T, int KB>
__global__ void __launch_bounds__(32) verify_words_kernel(const uint8_t *A, const uint8_t *B, const uint8_t *U,
                                                           const uint32_t *RB, const uint32_t *__restrict__ tabs,
                                                           int N, int K, int kblocks, int kw, size_t M, size_t batch,
                                                           unsigned long long *mismatch)
{
    const size_t Mw = M / 4;
    const size_t chunks = (Mw + 32 * kVwW - 1) / (32 * kVwW);
    // one warp per CTA: the unit index, the generation, the row addresses and
    // the r_jk masks are then CTA-uniform (uniform registers, not per-lane work)
    const size_t unit = blockIdx.x;
    if (unit >= batch * chunks) return;
    const int lane = threadIdx.x & 31;
    const size_t g = unit / chunks;
    const size_t w0 = (unit - g * chunks) * (32 * kVwW) + (size_t)lane;
    const uint32_t *Ag = reinterpret_cast<const uint32_t *>(A + g * (size_t)N * M) + w0;
    const uint32_t *Bg = reinterpret_cast<const uint32_t *>(B + g * (size_t)K * M) + w0;
    bool ok[kVwW];
#pragma unroll
    for (int v = 0; v < kVwW; v++) ok[v] = w0 + 32 * v < Mw;
    uint32_t bad = 0;
    for (int b0 = 0; b0 < kblocks; b0 += KB) {
        const int nb = min(KB, kblocks - b0);                  // blocks of this pass
        uint32_t y1[KB][T][kVwW];
#pragma unroll
        for (int bb = 0; bb < KB; bb++)
#pragma unroll
            for (int j = 0; j < T; j++)
#pragma unroll
                for (int v = 0; v < kVwW; v++) y1[bb][j][v] = 0u;
        const uint8_t *Ub = U + (g * kblocks + b0) * 2 * (size_t)N;   // block b0 + bb at Ub + 2 N bb
        // source words of four sources in flight while two are multiplied
        // (HBM latency, not issue, bounds a warp that waits per source)
        auto load2 = [&](int i, uint32_t (&a)[2][kVwW]) {
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
                for (int v = 0; v < kVwW; v++)
                    a[h][v] = (ok[v] && i + h < N) ? __ldg(Ag + (size_t)(i + h) * Mw + 32 * v) : 0u;
        };
        uint32_t acur[2][kVwW], anext[2][kVwW];
        load2(0, acur);
        load2(2, anext);
#pragma unroll 1
        for (int i = 0; i < N; i += 2) {
            uint32_t afar[2][kVwW];
            load2(i + 4, afar);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                if (i + h >= N) break;
                Sel sv[kVwW];
#pragma unroll
                for (int v = 0; v < kVwW; v++) sv[v] = make_sel(acur[h][v]);
#pragma unroll
                for (int bb = 0; bb < KB; bb++) {
                    if (bb >= nb) break;
#pragma unroll
                    for (int j = 0; j < T; j++) {
                        const uint32_t *tp = tabs + (size_t)__ldg(Ub + (size_t)(2 * bb + j) * N + i + h) * 16u;
                        const uint4 t0 = __ldg(reinterpret_cast<const uint4 *>(tp));
                        PrmtTab Tt;
                        Tt.t0lo = t0.x; Tt.t0hi = t0.y; Tt.t1lo = t0.z; Tt.t1hi = t0.w;
                        Tt.t2 = __ldg(tp + 4);
#pragma unroll
                        for (int v = 0; v < kVwW; v++) y1[bb][j][v] ^= lookup_perm(Tt, sv[v]);
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++)
#pragma unroll
                for (int v = 0; v < kVwW; v++) {
                    acur[h][v] = anext[h][v];
                    anext[h][v] = afar[h][v];
                }
        }
        // each block's coded rows eight at a time; a row in no projection is not read
#pragma unroll
        for (int bb = 0; bb < KB; bb++) {
            if (bb >= nb) break;
            const int b = b0 + bb;
            uint32_t y2[T][kVwW];
#pragma unroll
            for (int j = 0; j < T; j++)
#pragma unroll
                for (int v = 0; v < kVwW; v++) y2[j][v] = 0u;
            const int k1 = min(K, 64 * b + 64);
#pragma unroll 1
            for (int k0 = 64 * b; k0 < k1; k0 += 8) {
                uint32_t rb[T];
#pragma unroll
                for (int j = 0; j < T; j++) rb[j] = __ldg(RB + (g * 2 + j) * kw + (k0 >> 5)) >> (k0 & 31);   // 8 | 32
                uint32_t x[8][kVwW];
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    uint32_t sel = 0u;
#pragma unroll
                    for (int j = 0; j < T; j++) sel |= rb[j] >> e;
                    const bool need = (sel & 1u) && k0 + e < k1;
#pragma unroll
                    for (int v = 0; v < kVwW; v++)
                        x[e][v] = (need && ok[v]) ? __ldg(Bg + (size_t)(k0 + e) * Mw + 32 * v) : 0u;
                }
#pragma unroll
                for (int e = 0; e < 8; e++)
#pragma unroll
                    for (int j = 0; j < T; j++) {
                        const uint32_t m = 0u - ((rb[j] >> e) & 1u);
#pragma unroll
                        for (int v = 0; v < kVwW; v++) y2[j][v] ^= x[e][v] & m;
                    }
            }
#pragma unroll
            for (int j = 0; j < T; j++)
#pragma unroll
                for (int v = 0; v < kVwW; v++) bad += nz_bytes(unperm(y1[bb][j][v]) ^ y2[j][v]);
        }
    }
    const uint32_t nbad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && nbad) atomicAdd(mismatch + g, (unsigned long long)nbad);
}

// mismatch[g] += #{ positions where Y1[g] and Y2[g] differ }, Y: [batch][len]
__global__ void __launch_bounds__(256) count_mismatch_kernel(const uint8_t *Y1, const uint8_t *Y2, size_t len,
                                                             unsigned long long *mismatch)
{
    const size_t g = blockIdx.y;
    const uint8_t *a = Y1 + g * len, *b = Y2 + g * len;
    unsigned long long n = 0;
    for (size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x; x < len; x += (size_t)gridDim.x * blockDim.x)
        n += a[x] != b[x];
    for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(mismatch + g, n);
}

}  // namespace gfr
