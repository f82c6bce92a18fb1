// encode_stream.cuh -- batched RLNC encode for few coded packets (K <= 4),
// the paper's own measurement shape (N = 16 source packets, K = 1 coded
// packet):
//
//   B[g][k][m] = sum_i C[g][i][k] * A[g][i][m]          (Eq. 2)
//
// With K = 1 the encode is a streaming reduction: every source byte is read
// once and multiplied once, so it is bound by HBM (17 bytes of traffic per 16
// source bytes for N = 16), not by arithmetic -- provided the multiply stays
// under ~12 ALU operations per 32-bit word at HBM speed.  One thread owns one
// 16-byte column chunk of one generation: it loads the chunks of eight (GF(2),
// GF(4)) or four source packets at a time (16-byte non-allocating loads, all
// in flight together),
// multiplies each by its coefficient and XORs into K accumulators.  Per-field
// word arithmetic (coefficient tables from gf_init's table of tables,
// L1-resident):
//   GF(2):   acc ^= a & M0                                 1 LOP3
//   GF(4):   the paper's imul (Alg. 2): 2 IMAD + 1 LOP3
//            (a & 0x55..)*c ^ ((a>>1) & 0x55..)*(x c)
//   GF(16):  imul on the four nibble bit planes: 4 IMAD + 3 IMAD.HI (FMA
//            pipe) + 4 AND + 1 LOP3 (measured 2-4% faster than the PRMT form
//            below with GF(16) tables, which the same kernel also supports)
//   GF(256): three byte-permute split tables over bit groups {0-2}, {3-5},
//            {6-7} (Alg. 1's shuffle): 3 AND + 3 PRMT + 1
//            LOP3 on the ALU pipe, 3 IMAD.HI (selector packing) on the FMA
//            pipe; results in PRMT byte order, un-permuted once per output word.
// Products of two sources are folded into an accumulator with one 3-input
// XOR (LOP3): 7.5 ALU operations per source word for GF(256).
// Grid-stride over (generation, chunk); packets of 512 B or more give
// warp-uniform coefficients (broadcast table loads).
#pragma once
#include <cstdint>

#include "gf_device.cuh"
#include "tables.h"

namespace gfr {

constexpr int kStThreads = 256;


struct StreamParams {
    const uint8_t *A;
    const uint8_t *C;
    uint8_t *B;
    const uint32_t *tabs;   // table of tables of the field (16 words per coefficient)
    size_t M16;             // chunks per packet (16-byte chunks, or 4-byte ones for word-aligned packets)
    size_t total;           // batch * chunks per packet (strided / wide2 kernels: batch * wblocks * 32 threads)
    size_t wblocks;         // strided kernel: (32 W)-word blocks per packet; wide2: 64-chunk blocks
    int N, K;
    uint32_t qmask;
};

__device__ __forceinline__ uint4 st_ld_stream(const uint4 *p)
{
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// c * x for one 32-bit word, e = the coefficient's table entry.  kBatch =
// source chunks loaded together (measured), even; kPair = fold the products
// of two sources into the accumulator with one 3-input XOR (PRMT lookups end
// in an XOR anyway; for the masked / imul forms pairing only raised register
// use: GF(2) 97% -> 93%, GF(4) 89% -> 86% of HBM on the same box).
template <int F> struct StreamOp;
template <> struct StreamOp<2> {
    static constexpr bool kPermuted = false;
    static constexpr bool kPair = false;
    static constexpr int kBatch = 8;
    struct E { uint32_t m0; };
    __device__ __forceinline__ static E entry(const uint32_t *t) { return E{__ldg(t + 5)}; }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e) { return x & e.m0; }
};
template <> struct StreamOp<4> {
    static constexpr bool kPermuted = false;
    static constexpr bool kPair = false;
    static constexpr int kBatch = 8;
    struct E { uint32_t p0, p1; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(t + 8));
        return E{v.x, v.y};
    }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e)
    {
        return ((x & 0x55555555u) * e.p0) ^ ((mul_hi(x, 1u << 31) & 0x55555555u) * e.p1);
    }
};
struct StreamImul16 {      // GF(16) imul on the nibble bit planes
    static constexpr bool kPermuted = false;
    static constexpr bool kPair = false;
    static constexpr int kBatch = 4;
    struct E { uint32_t p0, p1, p2, p3; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(t + 8));
        return E{v.x, v.y, v.z, v.w};
    }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e)
    {
        const uint32_t n0 = x & 0x11111111u, n1 = mul_hi(x, 1u << 31) & 0x11111111u;
        const uint32_t n2 = mul_hi(x, 1u << 30) & 0x11111111u, n3 = mul_hi(x, 1u << 29) & 0x11111111u;
        return (n0 * e.p0) ^ (n1 * e.p1) ^ (n2 * e.p2) ^ (n3 * e.p3);
    }
};
struct StreamPrmt {        // split-table PRMT lookups (GF(16), GF(256))
    static constexpr bool kPermuted = true;
    static constexpr bool kPair = true;
    static constexpr int kBatch = 4;
    struct E { PrmtTab T; };
    __device__ __forceinline__ static E entry(const uint32_t *t)
    {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(t));
        E e;
        e.T.t0lo = v.x; e.T.t0hi = v.y; e.T.t1lo = v.z; e.T.t1hi = v.w; e.T.t2 = __ldg(t + 4);
        return e;
    }
    __device__ __forceinline__ static uint32_t mul(uint32_t x, const E &e) { return lookup_perm(e.T, make_sel(x)); }
};
template <> struct StreamOp<16> : StreamImul16 {};
template <> struct StreamOp<256> : StreamPrmt {};      // (StreamPrmt also serves GF(16): tables.cpp)

__device__ __forceinline__ uint32_t st_xor3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// table entry of coefficient C[g][i][k] (0 past the last source: its chunk is 0 too)
__device__ __forceinline__ const uint32_t *st_tab(const StreamParams &p, const uint8_t *Cg, int i, int k)
{
    const uint32_t c = i < p.N ? (__ldg(Cg + (size_t)i * p.K + k) & p.qmask) : 0u;
    return p.tabs + (size_t)c * kTableWords;
}

// generic V-word chunks; used with V = 1 (4-byte chunks) for packets that are
// only word aligned (e.g. C1's M = 1500)
template <int V> __device__ __forceinline__ void st_load(uint32_t (&a)[V], const uint8_t *p)
{
    if constexpr (V == 4) {
        const uint4 v = st_ld_stream(reinterpret_cast<const uint4 *>(p));
        a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
    } else {
        a[0] = __ldg(reinterpret_cast<const uint32_t *>(p));
    }
}
template <int V> __device__ __forceinline__ void st_store(uint8_t *p, const uint32_t (&r)[V])
{
    if constexpr (V == 4) *reinterpret_cast<uint4 *>(p) = make_uint4(r[0], r[1], r[2], r[3]);
    else *reinterpret_cast<uint32_t *>(p) = r[0];
}

// 16-byte chunks (packets 16-byte aligned): the measured fast form, kept as
// written for uint4 (a generic word-array version of it measured 2-6% slower)
template <class Op, int KT>
__global__ void __launch_bounds__(kStThreads) encode_stream_kernel(StreamParams p)
{
    constexpr int kStBatch = Op::kBatch;
    const size_t stride = (size_t)gridDim.x * kStThreads;
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t g = t / p.M16, ch = t - g * p.M16;
        const uint4 *Ag = reinterpret_cast<const uint4 *>(p.A + g * (size_t)p.N * (p.M16 * 16)) + ch;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint4 acc[KT];
#pragma unroll
        for (int k = 0; k < KT; k++) acc[k] = make_uint4(0u, 0u, 0u, 0u);
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint4 a[kStBatch];
#pragma unroll
            for (int b = 0; b < kStBatch; b++)
                a[b] = i0 + b < p.N ? st_ld_stream(Ag + (size_t)(i0 + b) * p.M16) : make_uint4(0u, 0u, 0u, 0u);
            if constexpr (Op::kPair) {
#pragma unroll
                for (int b = 0; b < kStBatch; b += 2) {
                    if (i0 + b >= p.N) break;
#pragma unroll
                    for (int k = 0; k < KT; k++) {
                        if (k < p.K) {
                            const typename Op::E e0 = Op::entry(st_tab(p, Cg, i0 + b, k));
                            const typename Op::E e1 = Op::entry(st_tab(p, Cg, i0 + b + 1, k));
                            acc[k].x = st_xor3(acc[k].x, Op::mul(a[b].x, e0), Op::mul(a[b + 1].x, e1));
                            acc[k].y = st_xor3(acc[k].y, Op::mul(a[b].y, e0), Op::mul(a[b + 1].y, e1));
                            acc[k].z = st_xor3(acc[k].z, Op::mul(a[b].z, e0), Op::mul(a[b + 1].z, e1));
                            acc[k].w = st_xor3(acc[k].w, Op::mul(a[b].w, e0), Op::mul(a[b + 1].w, e1));
                        }
                    }
                }
            } else {
#pragma unroll
                for (int b = 0; b < kStBatch; b++) {
                    if (i0 + b >= p.N) break;
#pragma unroll
                    for (int k = 0; k < KT; k++) {
                        if (k < p.K) {
                            const typename Op::E e = Op::entry(st_tab(p, Cg, i0 + b, k));
                            acc[k].x ^= Op::mul(a[b].x, e);
                            acc[k].y ^= Op::mul(a[b].y, e);
                            acc[k].z ^= Op::mul(a[b].z, e);
                            acc[k].w ^= Op::mul(a[b].w, e);
                        }
                    }
                }
            }
        }
        uint4 *Bg = reinterpret_cast<uint4 *>(p.B + g * (size_t)p.K * (p.M16 * 16)) + ch;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
                uint4 r = acc[k];
                if (Op::kPermuted) r = make_uint4(unperm(r.x), unperm(r.y), unperm(r.z), unperm(r.w));
                Bg[(size_t)k * p.M16] = r;
            }
        }
    }
}

template <class Op, int KT, int V>
__global__ void __launch_bounds__(kStThreads) encode_stream_words_kernel(StreamParams p)
{
    // 4-byte chunks: all 16 sources of a chunk in flight at once (one memory
    // latency per chunk instead of four: C1, one generation, is latency-bound)
    constexpr int kStBatch = V == 1 ? 16 : Op::kBatch;
    constexpr size_t kChunk = 4 * V;                           // bytes per chunk
    const size_t Mc = p.M16;                                   // chunks per packet
    const size_t M = Mc * kChunk;
    const size_t stride = (size_t)gridDim.x * kStThreads;
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t g = t / Mc, ch = t - g * Mc;
        const uint8_t *Ag = p.A + g * (size_t)p.N * M + ch * kChunk;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint32_t acc[KT][V];
#pragma unroll
        for (int k = 0; k < KT; k++)
#pragma unroll
            for (int v = 0; v < V; v++) acc[k][v] = 0u;
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint32_t a[kStBatch][V];
#pragma unroll
            for (int b = 0; b < kStBatch; b++) {
                if (i0 + b < p.N) st_load<V>(a[b], Ag + (size_t)(i0 + b) * M);
                else
#pragma unroll
                    for (int v = 0; v < V; v++) a[b][v] = 0u;
            }
#pragma unroll
            for (int b = 0; b < kStBatch; b += Op::kPair ? 2 : 1) {
                if (i0 + b >= p.N) break;
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    if (k < p.K) {
                        const typename Op::E e0 = Op::entry(st_tab(p, Cg, i0 + b, k));
                        if constexpr (Op::kPair) {
                            const typename Op::E e1 = Op::entry(st_tab(p, Cg, i0 + b + 1, k));
#pragma unroll
                            for (int v = 0; v < V; v++)
                                acc[k][v] = st_xor3(acc[k][v], Op::mul(a[b][v], e0), Op::mul(a[b + 1][v], e1));
                        } else {
#pragma unroll
                            for (int v = 0; v < V; v++) acc[k][v] ^= Op::mul(a[b][v], e0);
                        }
                    }
                }
            }
        }
        uint8_t *Bg = p.B + g * (size_t)p.K * M + ch * kChunk;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
                uint32_t r[V];
#pragma unroll
                for (int v = 0; v < V; v++) r[v] = Op::kPermuted ? unperm(acc[k][v]) : acc[k][v];
                st_store<V>(Bg + (size_t)k * M, r);
            }
        }
    }
}

// Word-aligned packets that are not 16-byte aligned (e.g. 1500 B) in bulk: a
// warp owns a block of 32 W consecutive words of one packet and lane l the
// words l, l + 32, ..., l + 32 (W - 1), so every 4-byte load instruction of the
// warp reads 128 contiguous bytes (full sectors); W (4, 8 or 12) is chosen per
// launch so that the blocks cover the packet well (1500 B = 375 words: one
// 384-word block, W = 12), and every per-source cost (coefficient byte, table
// entry, addresses) is paid once per W words.
template <class Op, int KT, int W>
__global__ void __launch_bounds__(kStThreads) encode_stream_strided_kernel(StreamParams p)
{
    constexpr int kStBatch = Op::kBatch;
    const size_t Mw = p.M16;                                   // words per packet
    const size_t M = Mw * 4;
    const size_t stride = (size_t)gridDim.x * kStThreads;     // a multiple of 32: t & 31 is the lane
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t blk = t >> 5;
        const size_t g = blk / p.wblocks;
        const size_t w0 = (blk - g * p.wblocks) * (32 * W) + (t & 31);
        bool ok[W];
#pragma unroll
        for (int j = 0; j < W; j++) ok[j] = w0 + 32 * j < Mw;
        const uint32_t *Ag = reinterpret_cast<const uint32_t *>(p.A + g * (size_t)p.N * M) + w0;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint32_t acc[KT][W];
#pragma unroll
        for (int k = 0; k < KT; k++)
#pragma unroll
            for (int j = 0; j < W; j++) acc[k][j] = 0u;
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint32_t a[kStBatch][W];
#pragma unroll
            for (int b = 0; b < kStBatch; b++)
#pragma unroll
                for (int j = 0; j < W; j++)
                    a[b][j] = (i0 + b < p.N && ok[j]) ? __ldg(Ag + (size_t)(i0 + b) * Mw + 32 * j) : 0u;
#pragma unroll
            for (int b = 0; b < kStBatch; b += Op::kPair ? 2 : 1) {
                if (i0 + b >= p.N) break;
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    if (k < p.K) {
                        const typename Op::E e0 = Op::entry(st_tab(p, Cg, i0 + b, k));
                        if constexpr (Op::kPair) {
                            const typename Op::E e1 = Op::entry(st_tab(p, Cg, i0 + b + 1, k));
#pragma unroll
                            for (int j = 0; j < W; j++)
                                acc[k][j] = st_xor3(acc[k][j], Op::mul(a[b][j], e0), Op::mul(a[b + 1][j], e1));
                        } else {
#pragma unroll
                            for (int j = 0; j < W; j++) acc[k][j] ^= Op::mul(a[b][j], e0);
                        }
                    }
                }
            }
        }
        uint32_t *Bg = reinterpret_cast<uint32_t *>(p.B + g * (size_t)p.K * M) + w0;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
#pragma unroll
                for (int j = 0; j < W; j++)
                    if (ok[j]) Bg[(size_t)k * Mw + 32 * j] = Op::kPermuted ? unperm(acc[k][j]) : acc[k][j];
            }
        }
    }
}

// 16-byte chunks, W (2 or 4) per thread (chunks l, l + 32, ... of a warp's
// (32 W)-chunk block of one packet): every per-source cost (coefficient byte,
// table entry, addresses) is paid once per 16 W source bytes instead of 16.
template <class Op, int KT, int W>
__global__ void __launch_bounds__(kStThreads) encode_stream_wide2_kernel(StreamParams p)
{
    constexpr int kStBatch = Op::kBatch;
    const size_t M16 = p.M16;
    const size_t stride = (size_t)gridDim.x * kStThreads;     // a multiple of 32: t & 31 is the lane
    for (size_t t = (size_t)blockIdx.x * kStThreads + threadIdx.x; t < p.total; t += stride) {
        const size_t blk = t >> 5;
        const size_t g = blk / p.wblocks;
        const size_t c0 = (blk - g * p.wblocks) * (32 * W) + (t & 31);
        bool ok[W];
#pragma unroll
        for (int j = 0; j < W; j++) ok[j] = c0 + 32 * j < M16;
        const uint4 *Ag = reinterpret_cast<const uint4 *>(p.A + g * (size_t)p.N * (M16 * 16)) + c0;
        const uint8_t *Cg = p.C + g * (size_t)p.N * p.K;
        uint4 acc[KT][W];
#pragma unroll
        for (int k = 0; k < KT; k++)
#pragma unroll
            for (int j = 0; j < W; j++) acc[k][j] = make_uint4(0u, 0u, 0u, 0u);
        for (int i0 = 0; i0 < p.N; i0 += kStBatch) {
            uint4 a[kStBatch][W];
#pragma unroll
            for (int b = 0; b < kStBatch; b++)
#pragma unroll
                for (int j = 0; j < W; j++)
                    a[b][j] = (i0 + b < p.N && ok[j]) ? st_ld_stream(Ag + (size_t)(i0 + b) * M16 + 32 * j)
                                                      : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int b = 0; b < kStBatch; b += Op::kPair ? 2 : 1) {
                if (i0 + b >= p.N) break;
#pragma unroll
                for (int k = 0; k < KT; k++) {
                    if (k < p.K) {
                        const typename Op::E e0 = Op::entry(st_tab(p, Cg, i0 + b, k));
                        if constexpr (Op::kPair) {
                            const typename Op::E e1 = Op::entry(st_tab(p, Cg, i0 + b + 1, k));
#pragma unroll
                            for (int j = 0; j < W; j++) {
                                acc[k][j].x = st_xor3(acc[k][j].x, Op::mul(a[b][j].x, e0), Op::mul(a[b + 1][j].x, e1));
                                acc[k][j].y = st_xor3(acc[k][j].y, Op::mul(a[b][j].y, e0), Op::mul(a[b + 1][j].y, e1));
                                acc[k][j].z = st_xor3(acc[k][j].z, Op::mul(a[b][j].z, e0), Op::mul(a[b + 1][j].z, e1));
                                acc[k][j].w = st_xor3(acc[k][j].w, Op::mul(a[b][j].w, e0), Op::mul(a[b + 1][j].w, e1));
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < W; j++) {
                                acc[k][j].x ^= Op::mul(a[b][j].x, e0); acc[k][j].y ^= Op::mul(a[b][j].y, e0);
                                acc[k][j].z ^= Op::mul(a[b][j].z, e0); acc[k][j].w ^= Op::mul(a[b][j].w, e0);
                            }
                        }
                    }
                }
            }
        }
        uint4 *Bg = reinterpret_cast<uint4 *>(p.B + g * (size_t)p.K * (M16 * 16)) + c0;
#pragma unroll
        for (int k = 0; k < KT; k++) {
            if (k < p.K) {
#pragma unroll
                for (int j = 0; j < W; j++) {
                    if (!ok[j]) continue;
                    uint4 r = acc[k][j];
                    if (Op::kPermuted) r = make_uint4(unperm(r.x), unperm(r.y), unperm(r.z), unperm(r.w));
                    Bg[(size_t)k * M16 + 32 * j] = r;
                }
            }
        }
    }
}

}  // namespace gfr
